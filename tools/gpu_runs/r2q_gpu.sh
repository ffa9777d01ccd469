python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/r2q_gputest.log 2>&1; tail -3 gpurun_out/r2q_gputest.log
for c in C2 C3; do timeout 300 python tools/pass2_probe.py $c 30 2>&1 | head -1; done
for c in C4 C5; do python bench.py --config $c --no-cpu-baseline --also none --steps 20 > gpurun_out/r2q_bench_$c.json 2> gpurun_out/r2q_bench_$c.err; tail -2 gpurun_out/r2q_bench_$c.err; done
