mkdir -p gpurun_out
timeout 600 python tools/e2e_loop_breakdown.py 20 > gpurun_out/e2e_breakdown.log 2>&1
cat gpurun_out/e2e_breakdown.log
nproc; lscpu | grep -i "model name\|socket\|numa node(s)"
