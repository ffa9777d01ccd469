for c in C2 C3 C4; do
python tools/step_probe.py $c tools/libdvl_old.so 40
python tools/step_probe.py $c tools/libdvl_new.so 40
done
