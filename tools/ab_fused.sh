# A/B timing of fused-kernel builds: bash tools/ab_fused.sh "variants" lib1.so lib2.so ...
# (the in-tree build is "cur"; variants are tools/time_fused.py variant ids)
V=${1:-1}; shift
for i in 1 2; do
  for l in "$@" cur; do
    if [ "$l" = cur ]; then python tools/time_fused.py 0 $V | sed "s/^/cur  /"
    else TSG_LIBRARY=$PWD/$l python tools/time_fused.py 0 $V | sed "s|^|$l  |"; fi
  done
done
