for l in build_ab/libtsg_peer.so cur; do
  if [ "$l" = cur ]; then unset TSG_LIBRARY; else export TSG_LIBRARY=$PWD/$l; fi
  timeout 300 python tools/bench_stencils.py ab 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('$l'.ljust(26), d['name'].ljust(30), str(d['patch']).ljust(16), '%8.1f us %5.1f%%' % (d['us'], 100*d['frac']))
    except Exception: pass
" | grep -E "cell_div|mpdata"
done
