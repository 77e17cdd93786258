for c in cfg2 cfg3; do python tools/kbench.py --config $c --mode full; python tools/kbench.py --config $c --mode full --pre; echo -n "$c "; python tools/prof_vcycle.py $c 2>&1 | grep -i replay; done
for p in 4 6 12 16; do echo -n "Q=$p "; PFFMG_Q2_ROWS=$p python tools/kbench.py --config cfg3 --mode full; done
