for c in C2 C3 C4; do
python tools/step_probe.py $c paper_2306_11612_b200/libdvl.so 40 write
python tools/step_probe.py $c paper_2306_11612_b200/libdvl.so 40 write+read
done
