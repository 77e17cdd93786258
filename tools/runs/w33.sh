timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/w33_base_tests.log 2>&1; echo "rc=$?" >> gpurun_out/w33_base_tests.log
bash tools/var/run.sh "--config cfg2 --mode full --reps 300" "--config cfg2 --mode chebbd --pre --reps 200" "--config cfg2 --mode resid --reps 200" "--config cfg2 --mode u --reps 200" "--config cfg2 --mode phi --reps 200" > gpurun_out/w33_var.txt 2>&1
LIB=paper_1902_08112_b200/libpffmg.so
cp $LIB /tmp/lib_orig.so
cp tools/var/lib_w33.so $LIB
python tools/prof_vcycle.py cfg2 2>/dev/null | head -1 > gpurun_out/w33_vc.txt
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_multigrid.py tests/test_gpu_configs.py tests/test_gpu_miehe.py tests/test_gpu_phi_table.py -x -q > gpurun_out/w33_tests.log 2>&1; echo "rc=$?" >> gpurun_out/w33_tests.log
cp /tmp/lib_orig.so $LIB
python tools/prof_vcycle.py cfg2 2>/dev/null | head -1 >> gpurun_out/w33_vc.txt
