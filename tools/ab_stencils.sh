# A/B of the secondary kernels between library builds on one box:
#   bash tools/ab_stencils.sh "regex" lib1.so lib2.so ...   ("cur" = the in-tree build)
PAT=${1:-.}; shift
for l in "$@" cur; do
  if [ "$l" = cur ]; then unset TSG_LIBRARY; else export TSG_LIBRARY=$PWD/$l; fi
  timeout 300 python tools/bench_stencils.py ab 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('$l'.ljust(24), d['name'].ljust(30), str(d['patch']).ljust(16), '%8.1f us %5.1f%%' % (d['us'], 100*d['frac']))
    except Exception: pass
" | grep -E "$PAT"
done
