# Round-end evidence from ONE source state: GPU tests, bench line, launch list,
# one ncu --set full capture of each config's vmult kernel, summarised ON the
# box with tools/ncu_summary.py (profiles/ncu_vmult_<cfg>_<TAG>.{json,md},
# copied into gpurun_out/; the large .ncu-rep files stay behind except cfg2's).
TAG=${1:-r2}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/cap_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/cap_gputests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/cap_bench.json 2> gpurun_out/cap_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/cap_bench_ref.json 2> gpurun_out/cap_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cap_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --extra "" > gpurun_out/cap_ncu_launch.log 2>&1
SHA=$(python -c "import bench; print(bench.src_sha())")
cap() {   # cfg kernel-regex command...
  local cfg=$1 k=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k $NCU_EXTRA -c 1 -o /tmp/cap_$cfg "$@" > gpurun_out/cap_$cfg.log 2>&1
  python tools/ncu_summary.py --rep /tmp/cap_$cfg.ncu-rep --name vmult_${cfg}_$TAG --src-sha $SHA \
    ${LAUNCHES:+--launches $LAUNCHES} ${BENCH:+--bench $BENCH} \
    --note "round-end capture (tools/runs/capture.sh): $*" >> gpurun_out/cap_summary.log 2>&1
  cp profiles/ncu_vmult_${cfg}_$TAG.json profiles/ncu_vmult_${cfg}_$TAG.md gpurun_out/ 2>/dev/null
  ncu -i /tmp/cap_$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/cap_${cfg}_sass.csv 2>/dev/null
}
LAUNCHES=gpurun_out/cap_launches.csv BENCH=gpurun_out/cap_bench.json NCU_EXTRA="--launch-skip 6" \
  cap cfg2 op2dw_kernel python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --extra ""
cp /tmp/cap_cfg2.ncu-rep gpurun_out/
cap cfg3 op2qs_kernel python tools/kbench.py --config cfg3 --mode full --reps 1
cap cfg4 op3dt_kernel python tools/kbench.py --config cfg4 --mode full --reps 1
cap cfg5 op3dt_kernel python tools/kbench.py --config cfg5 --mode full --reps 1
ls -la gpurun_out | grep cap_
