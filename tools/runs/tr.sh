# A/B: component-parallel restriction (2D levels up to PFFMG_RESTRICT_CP_MAXV vertices) + loads-first prolongation
LIB=paper_1902_08112_b200/libpffmg.so
cp $LIB /tmp/lib_orig.so
cp tools/var/lib_base.so $LIB
for c in cfg1 cfg2 cfg3 cfg4; do echo "== base $c $(python tools/prof_vcycle.py $c 2>/dev/null | head -1)"; done
cp tools/var/lib_tr.so $LIB
for m in 0 32768 131072 1000000; do
  export PFFMG_RESTRICT_CP_MAXV=$m
  for c in cfg1 cfg2; do echo "== tr maxv=$m $c $(python tools/prof_vcycle.py $c 2>/dev/null | head -1)"; done
done
unset PFFMG_RESTRICT_CP_MAXV
for c in cfg3 cfg4; do echo "== tr $c $(python tools/prof_vcycle.py $c 2>/dev/null | head -1)"; done
python tools/transferbench.py 2>&1 | grep "^=="
timeout 900 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_slabs.py tests/test_gpu_dist_solver.py tests/test_gpu_q2.py -m gpu -x -q 2>&1 | tail -2
cp /tmp/lib_orig.so $LIB
