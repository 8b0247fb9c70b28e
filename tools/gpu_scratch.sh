bash tools/gpu_round.sh > gpurun_out/round2.log 2>&1
cp gpurun_out/bench.log gpurun_out/bench_r2f.log; cp gpurun_out/bench_ref.log gpurun_out/bench_ref_r2f.log
grep -E "passed|failed|error" gpurun_out/gputest.log | tail -2; tail -1 gpurun_out/smoke.log
python tools/bench_brief.py gpurun_out/bench.log
tail -c 400 gpurun_out/bench_ref.log; echo; tail -c 300 gpurun_out/bench2.log
