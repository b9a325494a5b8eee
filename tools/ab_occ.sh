for k in 1 2 3; do
  libs="ablib/r02w.so ablib/occ_up.so"; [ $k != 1 ] && libs="$libs ablib/occ_dn.so"
  bash tools/ab_libs.sh $k $libs
done
