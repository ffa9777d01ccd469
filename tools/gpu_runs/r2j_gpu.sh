python tools/dist_probe.py 2 auto torch 2>&1 | tail -8
python tools/dist_probe.py 2 auto own 2>&1 | tail -8
python tools/dist_probe.py 2 lsd own 2>&1 | tail -8
python tools/dist_probe.py 1 auto own 2>&1 | tail -8
python tools/dist_probe.py 3 auto own 2>&1 | tail -8
