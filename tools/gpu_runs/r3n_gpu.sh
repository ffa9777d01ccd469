ncu --set full --clock-control none --import-source on -k regex:bin_boundary -s 6 -c 1 -o gpurun_out/r3n_bb_C3 python tools/edit_probe.py C3 10 > gpurun_out/r3n_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:agg_reduce -s 6 -c 1 -o gpurun_out/r3n_agg_C2 python tools/edit_probe.py C2 10 >> gpurun_out/r3n_ncu.log 2>&1
ls -la gpurun_out | grep r3n
