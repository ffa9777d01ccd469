free -g > gpurun_out/r2b_free.txt; nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> gpurun_out/r2b_free.txt
python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2b_gputest.log 2>&1; tail -25 gpurun_out/r2b_gputest.log
bash tools/sanitize.sh
python bench.py > gpurun_out/r2b_bench_C2.json 2> gpurun_out/r2b_bench_C2.err; tail -c 300 gpurun_out/r2b_bench_C2.json
python bench.py --config C4 --no-cpu-baseline > gpurun_out/r2b_bench_C4.json 2> gpurun_out/r2b_bench_C4.err; tail -c 300 gpurun_out/r2b_bench_C4.json; tail -3 gpurun_out/r2b_bench_C4.err
python bench.py --config C5 --no-cpu-baseline > gpurun_out/r2b_bench_C5.json 2> gpurun_out/r2b_bench_C5.err; tail -c 300 gpurun_out/r2b_bench_C5.json; tail -3 gpurun_out/r2b_bench_C5.err
