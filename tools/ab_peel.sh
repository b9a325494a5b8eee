set -x
L=paper_2510_16172_b200/lib/libfermat_b200.so
python tools/ab_bits.py ablib/r02u.so $L 1,2,3 2>&1 | grep -v " 0 of" ; echo "main bits done"
python tools/ab_bits.py ablib/r02u.so ablib/peel15.so 1,5 2>&1 | grep -v " 0 of"; echo "peel15 bits done"
python tools/ab_bits.py ablib/r02u.so ablib/peelall.so 1,2,3,4,5 2>&1 | grep -v " 0 of"; echo "peelall bits done"
for k in 1 5; do bash tools/ab_libs.sh $k ablib/r02u.so $L ablib/peel15.so ablib/peelall.so; done
for k in 2 3 4; do bash tools/ab_libs.sh $k ablib/r02u.so $L ablib/peelall.so; done
