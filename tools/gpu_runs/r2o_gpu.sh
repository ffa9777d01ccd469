python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_dist_build.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r2o_gputest.log 2>&1; tail -3 gpurun_out/r2o_gputest.log
for c in C2 C3 C1; do timeout 300 python tools/pass2_probe.py $c 30; done
