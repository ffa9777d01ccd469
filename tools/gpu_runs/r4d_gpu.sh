timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for k in 1 2; do
python tools/step_probe.py C2 ab/old.so 60
python tools/step_probe.py C2 ab/new.so 60
done
python tools/step_probe.py C1 ab/old.so 60
python tools/step_probe.py C1 ab/new.so 60
python tools/step_probe.py Cpaper ab/old.so 60
python tools/step_probe.py Cpaper ab/new.so 60
