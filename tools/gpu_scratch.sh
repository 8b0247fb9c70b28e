timeout 300 python tools/pcie_probe.py
