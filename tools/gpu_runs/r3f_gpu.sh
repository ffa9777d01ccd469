# launch lists (serialised, per-launch DRAM bytes) of the edit-cache step at C2, C3, C4
for c in C2 C3 C4; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r3f_launches_$c.csv python tools/edit_probe.py $c 8 > /dev/null 2>&1
done
ls -la gpurun_out | grep r3f
