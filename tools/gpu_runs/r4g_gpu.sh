# the prologue launched programmatically dependent as well
for k in 1 2; do
python tools/step_probe.py C2 ab/old.so 60
python tools/step_probe.py C2 ab/new.so 60
done
python tools/step_probe.py C3 ab/old.so 30
python tools/step_probe.py C3 ab/new.so 30
cp ab/prof_pdl.so paper_2306_11612_b200/libdvl.so
DVL_DBG=4 python tools/timeline.py C2 1024 2>/dev/null | grep -v nan
