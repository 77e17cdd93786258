mkdir -p gpurun_out
for m in full u phi; do
python tools/kbench.py --config cfg4 --mode $m --pre
for p in 2 3 4 5 6 8 11 13 17 22 33; do echo -n "P=$p "; PFFMG_3D_PLANES=$p python tools/kbench.py --config cfg4 --mode $m --pre; done
done > gpurun_out/sweep_cfg4.txt 2>&1
for m in full u; do
python tools/kbench.py --config cfg5 --levels 7 --mode $m --pre
for p in 4 8 12 16 24 32; do echo -n "P=$p "; PFFMG_3D_PLANES=$p python tools/kbench.py --config cfg5 --levels 7 --mode $m --pre; done
done > gpurun_out/sweep_cfg5.txt 2>&1
