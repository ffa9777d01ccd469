# final measurement pass of round 2 (after the launch-count fix and agg_jobs forms): GPU tests, smoke, bench lines
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r4c_gputest.log 2>&1; tail -3 gpurun_out/r4c_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/r4c_bench_C2.json 2> gpurun_out/r4c_bench_C2.err; tail -1 gpurun_out/r4c_bench_C2.err
python bench.py --config C4 --no-cpu-baseline --also none > gpurun_out/r4c_bench_C4.json 2> gpurun_out/r4c_bench_C4.err
python bench.py --config C5 --no-cpu-baseline --also none > gpurun_out/r4c_bench_C5.json 2> gpurun_out/r4c_bench_C5.err
python bench.py --config C1 --no-cpu-baseline --also none > gpurun_out/r4c_bench_C1.json 2> gpurun_out/r4c_bench_C1.err
python bench.py --config Cpaper --no-cpu-baseline --also none > gpurun_out/r4c_bench_Cpaper.json 2> gpurun_out/r4c_bench_Cpaper.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r4c_bench_reference.json 2> gpurun_out/r4c_bench_reference.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 1 --sharded --steps 20 --warmup 3 --also none > gpurun_out/r4c_bench_sharded_n1.json 2> gpurun_out/r4c_bench_sharded_n1.err
du -sh gpurun_out
