timeout 900 python -m pytest tests/test_gpu_api.py -q -x -k "streamed" 2>&1 | tail -2
timeout 300 python tools/streamed_probe.py 2>&1 | tail -3
