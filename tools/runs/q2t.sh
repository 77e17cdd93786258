timeout 1200 python -m pytest tests/test_gpu_q2.py tests/test_gpu_phi_table.py tests/test_gpu_configs.py tests/test_gpu_slabs.py -x -q -k "q2 or cfg3 or phi" > gpurun_out/q2t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q2t_tests.log
bash tools/var/run.sh "--config cfg3 --mode full --reps 200" "--config cfg3 --mode chebbd --pre --reps 100" "--config cfg3 --mode phi --reps 100" "--config cfg3 --mode u --reps 100" > gpurun_out/q2t_var.txt 2>&1
python tools/prof_vcycle.py cfg3 2>/dev/null | head -1 > gpurun_out/q2t_vc.txt
