# final-ish measurement pass: bench lines, reference arm, ncu captures
python bench.py > gpurun_out/r2s_bench_C2.json 2> gpurun_out/r2s_bench_C2.err; tail -2 gpurun_out/r2s_bench_C2.err
python bench.py --config C4 --no-cpu-baseline --also none > gpurun_out/r2s_bench_C4.json 2> gpurun_out/r2s_bench_C4.err
python bench.py --config C5 --no-cpu-baseline --also none > gpurun_out/r2s_bench_C5.json 2> gpurun_out/r2s_bench_C5.err
python bench.py --config C1 --no-cpu-baseline --also none > gpurun_out/r2s_bench_C1.json 2> gpurun_out/r2s_bench_C1.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2s_bench_reference.json 2> gpurun_out/r2s_bench_reference.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 1 --sharded --steps 20 --warmup 3 --also none > gpurun_out/r2s_bench_sharded_n1.json 2> gpurun_out/r2s_bench_sharded_n1.err
for c in C2 C3; do
  ncu --set full --clock-control none --import-source on -k regex:weights_reduce_tma -s 14 -c 1 -o gpurun_out/r2s_p1_$c python tools/edit_probe.py $c 20 > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:agg_reduce -s 8 -c 1 -o gpurun_out/r2s_p2_$c python tools/edit_probe.py $c 12 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"encode_bucket|bucket_scatter|bucket_rank|gather_validate8" -c 4 -o gpurun_out/r2s_build_C2 python tools/build_probe.py C2 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches_C2.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --also none > /dev/null 2>&1
ls -la gpurun_out | grep r2s
