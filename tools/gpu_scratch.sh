timeout 600 python tools/reduce_variants.py 256 256 80 0,6,7,9 2>&1 | grep -v '"variant": 1[0-9]'
timeout 600 python tools/reduce_variants.py 128 128 80 0,6,7,9 2>&1 | grep "VV\|CV\|EV"
