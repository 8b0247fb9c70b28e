timeout 600 python tools/sustained_variants.py 3
