timeout 600 python -m pytest tests/test_c_abi_example.py -q -m gpu 2>&1 | tail -5
