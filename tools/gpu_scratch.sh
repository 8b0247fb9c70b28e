timeout 300 python tools/dma2d_probe.py
