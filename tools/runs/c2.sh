timeout 900 python -m pytest tests/test_gpu_cheb2.py tests/test_gpu_multigrid.py -x -q > gpurun_out/c2tests.log 2>&1; echo "rc=$?" >> gpurun_out/c2tests.log
for f in 1 0; do for c in cfg1 cfg2; do echo "== FUSED_PAIRS=$f $c"; PFFMG_FUSED_PAIRS=$f python tools/prof_vcycle.py $c 2>/dev/null | head -2; done; done > gpurun_out/c2vc.txt 2>&1
