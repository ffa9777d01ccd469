python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/r2r_gputest.log 2>&1; tail -2 gpurun_out/r2r_gputest.log
python bench.py --steps 50 --also none --no-cpu-baseline > gpurun_out/r2r_bench_C2.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2r_bench_C2.json').read().strip().splitlines()[-1]); print('C2', d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernels_ms'])"
