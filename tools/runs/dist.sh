timeout 1500 python -m pytest tests/test_gpu_dist_solver.py tests/test_gpu_slabs.py -x -q 2>&1 | tail -25
