python paper_2306_11612_b200/build.py --define=DVL_PROF > /dev/null 2>&1
for c in C2 C3; do DVL_DBG=4 python tools/p1_spread.py $c; done
