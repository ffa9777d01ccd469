python bench.py --config C5 --no-cpu-baseline --also none > gpurun_out/r3o_bench_C5.json 2> gpurun_out/r3o_bench_C5.err; tail -2 gpurun_out/r3o_bench_C5.err
python bench.py --config C4 --no-cpu-baseline --also none > gpurun_out/r3o_bench_C4.json 2> gpurun_out/r3o_bench_C4.err
python paper_2306_11612_b200/build.py --define=DVL_PROF > /dev/null 2>&1 || echo build failed
DVL_DBG=4 python tools/awprobe.py C5
