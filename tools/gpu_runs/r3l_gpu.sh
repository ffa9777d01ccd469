python paper_2306_11612_b200/build.py --define=DVL_PROF > /dev/null 2>&1 || echo build failed
DVL_DBG=4 python tools/awprobe.py C3
DVL_DBG=4 python tools/awprobe.py C2
python paper_2306_11612_b200/build.py --force > /dev/null 2>&1 || echo build failed
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for c in C2 C3 C4; do
python tools/step_probe.py $c ab/old.so 40
python tools/step_probe.py $c ab/new.so 40
done
