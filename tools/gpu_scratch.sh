timeout 900 python -m pytest tests/test_gpu_api.py -x -q -k "cell or tma_reduce" 2>&1 | tail -3
timeout 600 python tools/reduce_variants.py celldiv 1024 1024 80 0,17 2>&1 | grep -v "^$"
timeout 600 python tools/reduce_variants.py celldiv 512 512 137 0 2>&1 | grep -v "^$"
