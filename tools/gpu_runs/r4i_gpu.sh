# fused prologue (U0 inside pass 1): parity, then A/B timing
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for k in 1 2; do
python tools/step_probe.py C2 ab/old.so 60
python tools/step_probe.py C2 ab/new.so 60
done
python tools/step_probe.py C3 ab/old.so 30
python tools/step_probe.py C3 ab/new.so 30
python tools/step_probe.py C5 ab/old.so 20
python tools/step_probe.py C5 ab/new.so 20
python tools/step_probe.py Cpaper ab/old.so 40
python tools/step_probe.py Cpaper ab/new.so 40
