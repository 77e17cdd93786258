for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --no-cpu --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/all_$c.json
  python tools/prof_vcycle.py $c 2>/dev/null | grep replay > gpurun_out/vc_$c.txt
done
