# Q2 staged at 3 CTAs/SM + 3D 16x16 tiles: full GPU suite, A/B timings, counters
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_b.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_b.log
for S in 1 0; do
  for m in full chebbd phi u; do
    PFFMG_Q2_STAGED=$S python tools/kbench.py --config cfg3 --mode $m --reps 100 >> gpurun_out/q2bench_b$S.txt 2>&1
  done
done
for T in 16 32; do
for m in full chebbd phi u chebu; do
  PFFMG_3D_TX=$T python tools/kbench.py --config cfg4 --mode $m --reps 100 >> gpurun_out/c4bench_$T.txt 2>&1
  PFFMG_3D_TX=$T python tools/kbench.py --config cfg5 --levels 7 --mode $m --reps 30 >> gpurun_out/c4bench_$T.txt 2>&1
done
PFFMG_3D_TX=$T python tools/kbench.py --config cfg5 --mode full --reps 10 >> gpurun_out/c4bench_$T.txt 2>&1
done
M=gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
ncu --metrics $M --clock-control none -k regex:"op2qs" -c 1 --csv python tools/kbench.py --config cfg3 --mode full --reps 1 > gpurun_out/q2m_b.csv 2>/dev/null
for T in 16 32; do
PFFMG_3D_TX=$T ncu --metrics $M --clock-control none -k regex:"op3dt" -c 1 --csv python tools/kbench.py --config cfg4 --mode full --reps 1 > gpurun_out/c4m_$T.csv 2>/dev/null
done
ncu --set full --import-source on --clock-control none -k regex:"op3dt_kernel" -c 1 -o gpurun_out/prof_c4_16 python tools/kbench.py --config cfg4 --mode full --reps 1 > gpurun_out/c4prof16.log 2>&1
ls -la gpurun_out
