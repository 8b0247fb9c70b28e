timeout 900 python -m pytest tests/test_gpu_reference_api.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py -x -q 2>&1 | tail -2
timeout 900 python tools/flat_stages_probe.py 1024 1024 81 2>&1 | grep divergence
for sz in "2560 2576 137" "1024 1024 81" "279 256 79"; do timeout 900 python tools/indirect_step_probe.py $sz 2>&1 | tail -1; done
