timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/trig_tests.log 2>&1; echo "rc=$?" >> gpurun_out/trig_tests.log
LIB=paper_1902_08112_b200/libpffmg.so
cp $LIB /tmp/lib_orig.so
for v in notrig trig; do
  cp tools/var/lib_$v.so $LIB
  for c in cfg1 cfg2 cfg3 cfg4; do echo "== $v $c $(python tools/prof_vcycle.py $c 2>/dev/null | head -1)"; done
  python tools/kbench.py --config cfg2 --mode full --reps 200
  python bench.py --steps 20 --warmup 5 --no-cpu --extra cfg3,cfg4 > gpurun_out/trig_bench_$v.json 2>/dev/null
done
cp /tmp/lib_orig.so $LIB
