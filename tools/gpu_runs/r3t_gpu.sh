python paper_2306_11612_b200/build.py --define=DVL_PROF > /dev/null 2>&1 || echo build failed
TL_PASS2=jobs DVL_DBG=4 python tools/timeline.py C3 4096 2>/dev/null | grep -v nan
DVL_DBG=4 python tools/timeline.py C3 4096 2>/dev/null | grep -v nan
