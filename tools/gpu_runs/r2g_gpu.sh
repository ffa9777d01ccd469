ncu --set full --clock-control none --import-source on -k regex:"encode_bucket|bucket_scatter|bucket_rank|gather_validate8" -o gpurun_out/r2g_build_C3 python tools/build_probe.py C3 1 > gpurun_out/r2g_ncu.log 2>&1
echo done
