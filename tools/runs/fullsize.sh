timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "l7" 2>&1 | tail -5
