LIB=paper_1902_08112_b200/libpffmg.so
cp $LIB /tmp/lib_orig.so
for v in base noedge; do
  cp tools/var/lib_$v.so $LIB
  echo "== $v"
  python tools/kbench.py --config cfg5 --levels 7 --mode full --reps 20
  python tools/kbench.py --config cfg5 --levels 7 --mode full --reps 20 --noexact
  PFFMG_3D_PLANES=8 python tools/kbench.py --config cfg5 --levels 7 --mode full --reps 20
  PFFMG_3D_PLANES=8 python tools/kbench.py --config cfg5 --levels 7 --mode full --reps 20 --noexact
done
cp /tmp/lib_orig.so $LIB
