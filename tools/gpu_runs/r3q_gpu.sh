timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_build.py -x -q 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_scale.py -x -q 2>&1 | tail -4
for c in C3 C4 C5 C2; do
python tools/step_probe.py $c ab/old.so 30
python tools/step_probe.py $c ab/new.so 30
done
