mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_reference_api.py -x -q 2>&1 | tail -15
