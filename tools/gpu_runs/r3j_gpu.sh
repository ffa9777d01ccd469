python paper_2306_11612_b200/build.py --define=DVL_PROF > /dev/null 2>&1 || echo build failed
BT_STRIDE=2368 DVL_DBG=4 python tools/aggprobe.py C3 4096
DVL_DBG=4 python tools/aggprobe.py C2 1024
AGG_TWICE=1 DVL_DBG=4 python tools/aggprobe.py C2 1024
