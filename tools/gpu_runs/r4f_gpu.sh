# timing experiment: the step without its prologue kernel (pass 1 first; results wrong)
python tools/step_probe.py C2 ab/prof.so 60
DVL_DBG=16 python tools/step_probe.py C2 ab/prof.so 60
python tools/step_probe.py C2 ab/prof.so 60
DVL_DBG=16 python tools/step_probe.py C2 ab/prof.so 60
python tools/step_probe.py C3 ab/prof.so 30
DVL_DBG=16 python tools/step_probe.py C3 ab/prof.so 30
