# A/B timing of fused-kernel builds: bash tools/ab_fused.sh lib1.so lib2.so ... (in-tree build = "cur")
for i in 1 2 3; do
  for l in "$@" cur; do
    if [ "$l" = cur ]; then python tools/time_fused.py 0 1 | sed "s/^/cur  /"
    else TSG_LIBRARY=$PWD/$l python tools/time_fused.py 0 1 | sed "s|^|$l  |"; fi
  done
done
