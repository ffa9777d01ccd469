# live timeline and per-warp pass-2 phases at C3 / C4 (DVL_PROF build)
python paper_2306_11612_b200/build.py --define=DVL_PROF > /dev/null 2>&1 || echo build failed
DVL_DBG=4 python tools/timeline.py C3 4096
DVL_DBG=4 python tools/aggprobe.py C3 4096
DVL_DBG=4 python tools/timeline.py C2 1024
