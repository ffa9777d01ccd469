python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/r2f_gputest.log 2>&1; tail -3 gpurun_out/r2f_gputest.log
for c in C2 C3 C4 C5; do python tools/build_probe.py $c 3 | tail -1; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ingest|encode|scan_|bucket|gather|agg_build" --csv --log-file gpurun_out/r2f_build_C5.csv python tools/build_probe.py C5 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ingest|encode|scan_|bucket|gather|agg_build" --csv --log-file gpurun_out/r2f_build_C2.csv python tools/build_probe.py C2 1 > /dev/null 2>&1
echo done
