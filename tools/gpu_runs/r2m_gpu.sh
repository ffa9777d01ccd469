for c in C2 C3; do
ncu --set full --clock-control none --import-source on -k regex:"weights_reduce_tma|agg_reduce|tf_prologue|epilogue_kernel|bin_boundary" -s 8 -c 4 -o gpurun_out/r2m_edit_$c python tools/edit_probe.py $c 6 > gpurun_out/r2m_ncu_$c.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"weights_reduce_tma|agg_reduce|tf_prologue|epilogue_kernel|bin_boundary" --csv --log-file gpurun_out/r2m_launch_$c.csv python tools/edit_probe.py $c 12 > /dev/null 2>&1
done
echo done
