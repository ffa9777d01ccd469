timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_build.py tests/test_gpu_scale.py -x -q 2>&1 | tail -2
for c in C3 C4 C5; do python tools/pass2_probe.py $c 20 | grep "stream\|jobs"; done
