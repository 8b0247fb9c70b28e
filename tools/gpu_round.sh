# Round-end rehearsal on one GPU: the driver's GPU tiers (pytest -m gpu, smoke, both bench
# arms, a 2-rank bench sharing the GPU).  Logs land in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
TSG_SHARE_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench2.log 2>&1
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 "$f"; done
