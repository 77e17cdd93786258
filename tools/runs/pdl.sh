# A/B: symmetric-Gauss transposes (lib_sym vs lib_old) and the early PDL trigger
# (lib_symearly) with the setup graph's launches stream-ordered or not
# (PFFMG_SETUP_PDL).  Kernel times by ncu durations, V-cycle replays by CUDA
# events, Newton steps from bench.py.
LIB=paper_1902_08112_b200/libpffmg.so
cp $LIB /tmp/lib_orig.so
for v in old sym symearly; do
  cp tools/var/lib_$v.so $LIB
  for sp in 1 0; do
    if [ $v != symearly ] && [ $sp = 0 ]; then continue; fi
    export PFFMG_SETUP_PDL=$sp
    for c in cfg1 cfg2 cfg3 cfg4; do echo "== $v setup_pdl=$sp $c $(python tools/prof_vcycle.py $c 2>/dev/null | head -1)"; done
    python bench.py --steps 20 --warmup 5 --no-cpu --extra cfg3,cfg4 > gpurun_out/pdl_bench_${v}_$sp.json 2>/dev/null
    python - <<EOF
import json
d = json.loads(open("gpurun_out/pdl_bench_${v}_$sp.json").read().strip().splitlines()[-1])
s = d["solve"]
print("== $v setup_pdl=$sp cfg2 vmult %.2f us  setup %.2f ms gmres %.2f ms step %.2f ms its %d" % (
    d["ms_per_step"] * 1e3, s["setup_ms"], s["gmres_ms"], s["ms_per_newton_step"], s["gmres_iters"]))
for c, x in (d.get("configs") or {}).items():
    print("== $v setup_pdl=$sp %s vmult %.2f us  setup %.2f ms gmres %.2f ms step %.2f ms its %d" % (
        c, x["vmult_ms"] * 1e3, x["setup_ms"], x["gmres_ms"], x["newton_step_ms"], x["gmres_iters"]))
EOF
  done
done
unset PFFMG_SETUP_PDL
cp /tmp/lib_orig.so $LIB
# kernel durations (ncu), old vs sym
for v in old sym; do
  cp tools/var/lib_$v.so $LIB
  for args in "--config cfg2 --mode full" "--config cfg4 --mode full" "--config cfg5 --levels 7 --mode full" "--config cfg2 --mode chebbd --pre"; do
    K=op
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"op2dw|op3dt" --csv python tools/kbench.py $args --reps 12 2>/dev/null \
      | python -c "
import sys,csv
r=[x for x in csv.reader(sys.stdin) if len(x)>10 and x[-3]=='gpu__time_duration.sum']
d=[float(x[-1].replace(',','')) for x in r][3:]
print('== ncu $v', '$args', 'n=%d mean %.2f us min %.2f'%(len(d), sum(d)/len(d)/1e3, min(d)/1e3) if d else 'none')"
  done
done
cp /tmp/lib_orig.so $LIB
for c in cfg2 cfg4; do PFFMG_VC_SEQ=1 python tools/prof_vcycle.py $c > gpurun_out/vc_$c.txt 2>&1; done
python tools/prof_newton.py cfg2 > gpurun_out/newton_cfg2.txt 2>&1
