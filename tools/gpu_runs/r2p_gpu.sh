python -m pytest tests -m gpu -x -q > gpurun_out/r2p_gputest.log 2>&1; tail -3 gpurun_out/r2p_gputest.log
for c in C4 C5; do python bench.py --config $c --no-cpu-baseline --also none --steps 20 > gpurun_out/r2p_bench_$c.json 2> gpurun_out/r2p_bench_$c.err; tail -2 gpurun_out/r2p_bench_$c.err; done
