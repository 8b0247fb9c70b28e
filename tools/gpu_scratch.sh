for i in 1 2; do
echo base; timeout 300 python tools/sustained_variants.py 3 0
echo signflip; TSG_LIBRARY=$PWD/paper_1908_06094_b200/libtsg_sf.so timeout 300 python tools/sustained_variants.py 3 0
done
