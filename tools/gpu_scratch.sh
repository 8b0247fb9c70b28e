timeout 600 python tools/loop_paths_probe.py
