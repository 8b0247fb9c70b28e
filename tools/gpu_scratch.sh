timeout 900 python -m pytest tests/test_distributed.py -q -x -k "p2p_fused" 2>&1 | tail -3
