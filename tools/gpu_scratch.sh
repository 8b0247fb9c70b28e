timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_reference_api.py tests/test_gpu_acceptance.py -x -q -k "not long_sweeps" > gpurun_out/san_flat_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/san_flat_memcheck.log
timeout 900 compute-sanitizer --tool memcheck python tools/indirect_step_probe.py 37 45 21 2>&1 | tail -2
