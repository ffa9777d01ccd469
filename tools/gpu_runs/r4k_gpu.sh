# race check at size: bit-identical vertices across contexts and pass-2 forms
python tools/determinism_probe.py C2 60 auto,auto,list,jobs
python tools/determinism_probe.py C3 40 auto,auto,inline,jobs
python tools/determinism_probe.py C4 30 auto,auto,list
python tools/determinism_probe.py C5 20 auto,auto
