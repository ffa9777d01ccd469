for i in 1 2; do
python tools/step_probe.py C2 tools/libdvl_base.so 40
python tools/step_probe.py C2 tools/libdvl_nowait.so 40
done
