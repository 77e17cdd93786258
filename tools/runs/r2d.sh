# persistent 2D / Q2 / strip-major 3D: GPU suite, variant timings, bench, ncu
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_d.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_d.log
bash tools/var/run.sh "--config cfg3 --mode full --reps 100" "--config cfg3 --mode chebbd --pre --reps 100" "--config cfg3 --mode u --reps 100" > gpurun_out/q2var_d.txt 2>&1
for m in full chebbd phi u resid; do
  python tools/kbench.py --config cfg2 --mode $m --reps 200 >> gpurun_out/c2bench_d.txt 2>&1
done
python tools/kbench.py --config cfg2 --mode chebbd --pre --reps 200 >> gpurun_out/c2bench_d.txt 2>&1
for m in full chebbd phi u chebu; do
  python tools/kbench.py --config cfg4 --mode $m --reps 100 >> gpurun_out/c4bench_d.txt 2>&1
  python tools/kbench.py --config cfg5 --levels 7 --mode $m --reps 30 >> gpurun_out/c4bench_d.txt 2>&1
done
python tools/kbench.py --config cfg5 --mode full --reps 10 >> gpurun_out/c4bench_d.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
M=gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:"op2dw" -c 1 --csv python tools/kbench.py --config cfg2 --mode full --reps 1 > gpurun_out/c2m_d.csv 2>/dev/null
ncu --metrics $M --clock-control none -k regex:"op3dt" -c 1 --csv python tools/kbench.py --config cfg4 --mode full --reps 1 > gpurun_out/c4m_d.csv 2>/dev/null
ls -la gpurun_out
