# pass 2 with and without its accumulator atomics (DVL_PROF timing experiment)
python paper_2306_11612_b200/build.py --define=DVL_PROF > /dev/null 2>&1 || echo build failed
DVL_DBG=4 python tools/timeline.py C3 4096
DVL_DBG=4 TL_NORED=1 python tools/timeline.py C3 4096
DVL_DBG=4 python tools/timeline.py C2 1024
DVL_DBG=4 TL_NORED=1 python tools/timeline.py C2 1024
