for m in phi chebp u full; do python tools/kbench.py --config cfg4 --mode $m --pre; done
for p in 2 3 4 6 8 12; do echo -n "P=$p "; PFFMG_3D_PLANES=$p python tools/kbench.py --config cfg4 --mode chebp --pre; done
python tools/kbench.py --config cfg5 --levels 7 --mode chebp --pre
for p in 4 8 16 32; do echo -n "P=$p "; PFFMG_3D_PLANES=$p python tools/kbench.py --config cfg5 --levels 7 --mode chebp --pre; done
echo -n "cfg4 "; python tools/prof_vcycle.py cfg4 2>&1 | grep -i replay
