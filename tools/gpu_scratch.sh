timeout 900 python -m pytest tests/test_gpu_api.py -q -x -k "shared_divisor or cell_div or tma_reduce" 2>&1 | tail -4
timeout 300 python tools/celldiv_probe.py
