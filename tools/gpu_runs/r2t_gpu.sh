for c in C4 C2; do
python tools/step_probe.py $c tools/libdvl_prev.so 50
python tools/step_probe.py $c paper_2306_11612_b200/libdvl.so 50
python tools/step_probe.py $c tools/libdvl_prev.so 20
python tools/step_probe.py $c paper_2306_11612_b200/libdvl.so 20
done
