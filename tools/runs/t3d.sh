timeout 600 python -m pytest tests/test_gpu_operator.py -x -q -k "exact" 2>&1 | tail -3
for m in full u chebu; do
python tools/kbench.py --config cfg4 --mode $m --reps 50
python tools/kbench.py --config cfg4 --mode $m --reps 50 --noexact
done
