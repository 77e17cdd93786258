timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_g.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_g.log
bash tools/var/run.sh "--config cfg3 --mode full --reps 100" "--config cfg3 --mode chebbd --pre --reps 100" "--config cfg3 --mode phi --reps 100" "--config cfg3 --mode u --reps 100" > gpurun_out/q2var_g.txt 2>&1
for m in full chebbd phi u chebu; do
  python tools/kbench.py --config cfg4 --mode $m --reps 100 >> gpurun_out/bench_g.txt 2>&1
  python tools/kbench.py --config cfg5 --levels 7 --mode $m --reps 30 >> gpurun_out/bench_g.txt 2>&1
done
python tools/kbench.py --config cfg5 --mode full --reps 10 >> gpurun_out/bench_g.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:"op3dt_kernel" -c 1 -o gpurun_out/prof_c4_g python tools/kbench.py --config cfg4 --mode full --reps 1 > gpurun_out/c4prof_g.log 2>&1
