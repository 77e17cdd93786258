for c in cfg2 cfg3 cfg4; do python tools/prof_vcycle.py $c > gpurun_out/vc_$c.txt 2>&1; done
python tools/prof_gmres.py cfg2 > gpurun_out/gm_cfg2.txt 2>&1
