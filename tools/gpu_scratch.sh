for tool in memcheck synccheck; do
timeout 1800 compute-sanitizer --tool $tool python tools/sanitize_dyn.py 200x400x36 > gpurun_out/san_dyn_$tool.log 2>&1; echo "$tool rc=$?"; tail -1 gpurun_out/san_dyn_$tool.log
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
