# A/B of the O1280-class fused step between library builds on one box:
#   bash tools/ab_o1280.sh lib1.so lib2.so ...   ("cur" = the in-tree build)
for i in 1 2; do
  for l in "$@" cur; do
    if [ "$l" = cur ]; then unset TSG_LIBRARY; else export TSG_LIBRARY=$PWD/$l; fi
    python bench.py --workload o1280 --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1])
print('$l'.ljust(22), '%.3f ms' % d['ms_per_step'], '%.1f%%' % (100*d['roofline']['frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
