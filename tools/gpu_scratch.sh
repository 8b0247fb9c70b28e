timeout 900 python -m pytest tests/test_gpu_reference_api.py -x -q 2>&1 | tail -2
for sz in "1024 1024 81" "279 256 79"; do timeout 900 python tools/flat_stages_probe.py $sz 2>&1 | grep cell_div; done
