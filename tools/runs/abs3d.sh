# A/B: warp-uniform branch around the absent-cell select of the 3D tile kernel
bash tools/var/ncu_ab.sh "op3dt" "--config cfg4 --mode full" "--config cfg5 --levels 7 --mode full" "--config cfg5 --levels 7 --mode chebu --pre" "--config cfg4 --mode chebu --pre" "--config cfg5 --levels 7 --mode phi"
LIB=paper_1902_08112_b200/libpffmg.so
cp $LIB /tmp/lib_orig.so
for v in base abs; do
  cp tools/var/lib_$v.so $LIB
  echo "== $v cfg4 $(python tools/prof_vcycle.py cfg4 2>/dev/null | head -1)"
  python tools/kbench.py --config cfg5 --mode full --reps 20
done
cp /tmp/lib_orig.so $LIB
