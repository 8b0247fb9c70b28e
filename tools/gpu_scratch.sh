timeout 300 python tools/sustained_copy_probe.py 3 | tail -4
nvidia-smi --query-gpu=power.draw,power.limit --format=csv
