set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for c in C2 C3 C4; do
python tools/step_probe.py $c ab/old.so 40
python tools/step_probe.py $c ab/new.so 40
python tools/step_probe.py $c ab/old.so 40
python tools/step_probe.py $c ab/new.so 40
done
