python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gputest.log 2>&1; tail -5 gpurun_out/r2c_gputest.log
for c in C2 C5 C4; do python bench.py --config $c --no-cpu-baseline --also none --steps 20 > gpurun_out/r2c_bench_$c.json 2> gpurun_out/r2c_bench_$c.err; tail -3 gpurun_out/r2c_bench_$c.err; done
