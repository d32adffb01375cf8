for v in default u2 u4 u8 c1r4u8; do
  if [ $v = default ]; then unset S2W_LIB; else export S2W_LIB=$PWD/lib_var/$v/libs2w.so; fi
  echo "== $v"; python scripts/time_sht.py --L 2048 --scheme mw --reps 5 | grep analysis
  python scripts/time_sht.py --L 4096 --scheme mw --real --reps 3 | grep analysis
done
