# lean Chebyshev start (d-only x = 0 start + pffmg_cheb_first_*): tests, then V-cycle / Newton A/B
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/lean_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/lean_tests.log
for f in 1 0; do
  export PFFMG_LEAN_START=$f
  for c in cfg1 cfg2 cfg3 cfg4; do echo "== lean=$f $c $(python tools/prof_vcycle.py $c 2>/dev/null | head -1)"; done
  python bench.py --steps 20 --warmup 5 --no-cpu --extra cfg3,cfg4,cfg5 > gpurun_out/lean_bench_$f.json 2>/dev/null
  python - <<PY
import json
d = json.loads(open("gpurun_out/lean_bench_$f.json").read().strip().splitlines()[-1])
s = d["solve"]
print("== lean=$f cfg2 setup %.2f ms gmres %.2f ms step %.2f ms its %d" % (s["setup_ms"], s["gmres_ms"], s["ms_per_newton_step"], s["gmres_iters"]))
for c, x in (d.get("configs") or {}).items():
    print("== lean=$f %s setup %.2f ms gmres %.2f ms step %.2f ms its %d" % (c, x["setup_ms"], x["gmres_ms"], x["newton_step_ms"], x["gmres_iters"]))
PY
done
