# final measurement pass of round 2, part 2: ncu launch lists and full captures, summarised on
# the box (the .ncu-rep files stay there)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3w_launches_C2.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --also none > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/r3w_launches_C2.csv > gpurun_out/r3w_launches_C2.md
for c in C3 C4 C5; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file /tmp/l_$c.csv python tools/edit_probe.py $c 6 > /dev/null 2>&1
python tools/ncu_csv.py /tmp/l_$c.csv > gpurun_out/r3w_launches_edit_$c.md
done
mkdir -p /tmp/reps
for c in C2 C3; do
  ncu --set full --clock-control none --import-source on -k regex:weights_reduce_tma -s 14 -c 1 -o /tmp/reps/p1_$c python tools/edit_probe.py $c 20 > /dev/null 2>&1
  ncu -i /tmp/reps/p1_$c.ncu-rep --page raw --csv > /tmp/reps/p1_$c.csv
  python profiles/summarize_full.py /tmp/reps/p1_$c.csv > gpurun_out/r3w_ncu_full_p1_$c.md
done
ncu --set full --clock-control none --import-source on -k regex:agg_jobs -s 3 -c 1 -o /tmp/reps/p2_C5 python tools/edit_probe.py C5 6 > /dev/null 2>&1
ncu -i /tmp/reps/p2_C5.ncu-rep --page raw --csv > /tmp/reps/p2_C5.csv
python profiles/summarize_full.py /tmp/reps/p2_C5.csv > gpurun_out/r3w_ncu_full_agg_jobs_C5.md
ncu --set full --clock-control none --import-source on -k regex:bin_boundary -s 3 -c 1 -o /tmp/reps/bb_C3 python tools/edit_probe.py C3 6 > /dev/null 2>&1
ncu -i /tmp/reps/bb_C3.ncu-rep --page raw --csv > /tmp/reps/bb_C3.csv
python profiles/summarize_full.py /tmp/reps/bb_C3.csv > gpurun_out/r3w_ncu_full_bin_boundary_C3.md
du -sh gpurun_out; ls -la gpurun_out
