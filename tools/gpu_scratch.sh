timeout 600 python tools/op_sustained_o1280.py
