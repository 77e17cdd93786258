# persistent 3D kernel (+ tile list), Q2 flag fix: GPU suite, timings, ncu
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_c.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_c.log
for m in full chebbd phi u; do
  python tools/kbench.py --config cfg3 --mode $m --reps 100 >> gpurun_out/q2bench_c.txt 2>&1
done
for m in full chebbd phi u chebu; do
  python tools/kbench.py --config cfg4 --mode $m --reps 100 >> gpurun_out/c4bench_c.txt 2>&1
  python tools/kbench.py --config cfg5 --levels 7 --mode $m --reps 30 >> gpurun_out/c4bench_c.txt 2>&1
done
python tools/kbench.py --config cfg5 --mode full --reps 10 >> gpurun_out/c4bench_c.txt 2>&1
for C in 1 2; do
  PFFMG_3D_CTAS=$C python tools/kbench.py --config cfg4 --mode full --reps 100 >> gpurun_out/c4ctas.txt 2>&1
  PFFMG_3D_CTAS=$C python tools/kbench.py --config cfg4 --mode u --reps 100 >> gpurun_out/c4ctas.txt 2>&1
done
M=gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:"op2qs" -c 1 --csv python tools/kbench.py --config cfg3 --mode full --reps 1 > gpurun_out/q2m_c.csv 2>/dev/null
ncu --metrics $M --clock-control none -k regex:"op3dt" -c 1 --csv python tools/kbench.py --config cfg4 --mode full --reps 1 > gpurun_out/c4m_c.csv 2>/dev/null
ncu --metrics $M --clock-control none -k regex:"op3dt" -c 1 --csv python tools/kbench.py --config cfg5 --levels 7 --mode full --reps 1 > gpurun_out/c5m_c.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:"op2qs_kernel" -c 1 -o gpurun_out/prof_q2s_c python tools/kbench.py --config cfg3 --mode full --reps 1 > gpurun_out/q2prof_c.log 2>&1
ls -la gpurun_out
