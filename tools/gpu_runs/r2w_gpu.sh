python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dist_build.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -2
for c in C2 C3 C5; do python tools/build_probe.py $c 3 | tail -1; done
