python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dist_build.py -m gpu -x -q > gpurun_out/r2u_gputest.log 2>&1; tail -2 gpurun_out/r2u_gputest.log
python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q --durations=5 > gpurun_out/r2u_fullsize.log 2>&1; tail -12 gpurun_out/r2u_fullsize.log
python tools/step_probe.py C4 paper_2306_11612_b200/libdvl.so 30
for c in C2 C3 C5; do python tools/build_probe.py $c 3 | tail -1; done
