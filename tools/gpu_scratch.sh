CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_reference_api.py tests/test_gpu_acceptance.py "tests/test_gpu_api.py::test_pack_unpack_roundtrip_every_numbering" "tests/test_gpu_api.py::test_table1_kernels_direct_and_indirect" "tests/test_gpu_api.py::test_relabelled_flat_paths_are_invariant" "tests/test_gpu_api.py::test_indirect_reduce_every_width" -q -x > gpurun_out/memcheck_r2.log 2>&1
echo rc=$?
grep -v "^=========     \(#\|in \|Saved\)" gpurun_out/memcheck_r2.log | tail -8
