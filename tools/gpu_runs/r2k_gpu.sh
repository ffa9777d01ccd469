python -m pytest tests -m gpu -q > gpurun_out/r2k_gputest.log 2>&1; tail -3 gpurun_out/r2k_gputest.log
python bench.py > gpurun_out/r2k_bench_C2.json 2> gpurun_out/r2k_bench_C2.err; tail -3 gpurun_out/r2k_bench_C2.err
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
