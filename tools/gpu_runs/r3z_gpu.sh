python paper_2306_11612_b200/build.py --define=DVL_PROF > /dev/null 2>&1 || echo build failed
DVL_DBG=4 python tools/aggprobe.py C2 1024
