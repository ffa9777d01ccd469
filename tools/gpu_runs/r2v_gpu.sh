python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do python tools/step_probe.py C2 paper_2306_11612_b200/libdvl.so 50; done
python tools/step_probe.py C1 paper_2306_11612_b200/libdvl.so 50
