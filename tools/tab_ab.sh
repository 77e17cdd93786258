for m in full u chebu phi chebp; do python tools/kbench.py --config cfg4 --mode $m --pre; done
python tools/kbench.py --config cfg4 --mode full
echo -n "cfg4 "; python tools/prof_vcycle.py cfg4 2>&1 | grep -i replay
