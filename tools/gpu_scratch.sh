OLD=$PWD/paper_1908_06094_b200/libtsg_old.so
for i in 1 2; do
echo new; timeout 300 python tools/celldiv_probe.py
echo old; TSG_LIBRARY=$OLD timeout 300 python tools/celldiv_probe.py
done
