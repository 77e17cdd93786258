timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_f.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_f.log
for m in full chebbd phi u resid; do python tools/kbench.py --config cfg2 --mode $m --reps 200 >> gpurun_out/bench_f.txt 2>&1; done
for m in full chebbd phi u; do python tools/kbench.py --config cfg3 --mode $m --reps 100 >> gpurun_out/bench_f.txt 2>&1; done
for m in full chebbd phi u chebu; do
  python tools/kbench.py --config cfg4 --mode $m --reps 100 >> gpurun_out/bench_f.txt 2>&1
  python tools/kbench.py --config cfg5 --levels 7 --mode $m --reps 30 >> gpurun_out/bench_f.txt 2>&1
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
