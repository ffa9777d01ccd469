python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -1
for c in C2 C3 C4 C5; do python tools/step_probe.py $c paper_2306_11612_b200/libdvl.so 30; done
