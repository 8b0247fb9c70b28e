for rep in 1 2; do for lib in libtsg.so libtsg_d1.so; do echo "== $lib"
TSG_LIBRARY=$PWD/paper_1908_06094_b200/$lib timeout 600 python tools/flat_stages_probe.py 2>&1 | grep cell_div
TSG_LIBRARY=$PWD/paper_1908_06094_b200/$lib timeout 600 python tools/flat_stages_probe.py 279 256 80 2>&1 | grep cell_div
done; done
timeout 900 python -m pytest tests/test_gpu_reference_api.py -x -q 2>&1 | tail -2
