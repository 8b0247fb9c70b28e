timeout 900 python -m pytest tests/test_gpu_reference_api.py tests/test_gpu_api.py tests/test_gpu_parity.py -x -q -k "neighbor or table1 or flat or one_dim or relabel or reduce" 2>&1 | tail -2
for sz in "1024 1024 81" "1024 1024 80" "128 128 81"; do timeout 900 python tools/flat_stages_probe.py $sz 2>&1 | grep neighbor; done
