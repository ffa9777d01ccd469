python paper_2306_11612_b200/build.py --define=DVL_PROF > /dev/null 2>&1
DVL_DBG=4 python tools/timeline.py C2 2>&1 | tail -25
