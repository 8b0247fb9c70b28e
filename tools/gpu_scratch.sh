timeout 900 python -m pytest tests/test_gpu_api.py -q -x -k "many_launches" 2>&1 | tail -2
