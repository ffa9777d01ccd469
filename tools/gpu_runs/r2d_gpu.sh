python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sort or dup or c1 or amr or u64 or full" > gpurun_out/r2d_gputest.log 2>&1; tail -3 gpurun_out/r2d_gputest.log
for c in C2 C5 C4 C3; do python tools/build_probe.py $c 3; done
python tools/build_probe.py C2 2 lsd
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_build_C2.csv python tools/build_probe.py C2 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_build_C5.csv python tools/build_probe.py C5 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"bucket|encode_bucket|gather_validate4" -c 6 -o gpurun_out/r2d_build_C5 python tools/build_probe.py C5 1 > /dev/null 2>&1
echo done
