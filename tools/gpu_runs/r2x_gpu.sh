python -m pytest tests/test_gpu_locate.py tests/test_gpu_dist_build.py -m gpu -x -q 2>&1 | tail -3
