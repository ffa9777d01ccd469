timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for c in C2 C3 C4 C5 C2; do
python tools/step_probe.py $c ab/old.so 40
python tools/step_probe.py $c ab/new.so 40
done
