# staged Q2 kernel: parity tests, A/B timings, ncu of cfg3 FULL; cfg4 3D counters
timeout 900 python -m pytest tests/test_gpu_q2.py tests/test_gpu_configs.py -x -q -k "q2 or cfg3" > gpurun_out/q2tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/q2tests.log
for S in 1 0; do
  for m in full chebbd phi u resid; do
    PFFMG_Q2_STAGED=$S python tools/kbench.py --config cfg3 --mode $m --reps 100 >> gpurun_out/q2bench_$S.txt 2>&1
  done
  PFFMG_Q2_STAGED=$S python tools/kbench.py --config cfg3 --mode chebbd --pre --reps 100 >> gpurun_out/q2bench_$S.txt 2>&1
done
for m in full chebbd phi u; do
  python tools/kbench.py --config cfg4 --mode $m --reps 100 >> gpurun_out/c4bench.txt 2>&1
  python tools/kbench.py --config cfg5 --levels 7 --mode $m --reps 30 >> gpurun_out/c4bench.txt 2>&1
done
M=gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem
for S in 1 0; do
PFFMG_Q2_STAGED=$S ncu --metrics $M --clock-control none -k regex:"op2q" -c 2 --csv python tools/kbench.py --config cfg3 --mode full --reps 1 > gpurun_out/q2m_$S.csv 2>/dev/null
done
ncu --set full --import-source on --clock-control none -k regex:"op2qs_kernel" -c 1 -o gpurun_out/prof_q2s python tools/kbench.py --config cfg3 --mode full --reps 1 > gpurun_out/q2prof.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"op3dt_kernel" -c 1 -o gpurun_out/prof_c4 python tools/kbench.py --config cfg4 --mode full --reps 1 > gpurun_out/c4prof.log 2>&1
ls -la gpurun_out
