# A/B: warp-uniform branch around the absent-cell select of the 2D FULL kernels
bash tools/var/ncu_ab.sh "op2dw" "--config cfg2 --mode full" "--config cfg2 --mode chebbd --pre" "--config cfg2 --mode resid --pre" "--config cfg1 --mode full" "--config cfg2 --levels 7 --mode chebbd --pre"
LIB=paper_1902_08112_b200/libpffmg.so
cp $LIB /tmp/lib_orig.so
for v in base selb; do
  cp tools/var/lib_$v.so $LIB
  for c in cfg1 cfg2; do echo "== $v $c $(python tools/prof_vcycle.py $c 2>/dev/null | head -1)"; done
  python tools/kbench.py --config cfg2 --mode full --reps 300
done
cp /tmp/lib_orig.so $LIB
