timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "launch_count or edit_cache or sizes" 2>&1 | tail -3
python bench.py --config C5 --no-cpu-baseline --also none --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5 launches', d['gpu_launches'], d['steps'])"
python bench.py --config C3 --no-cpu-baseline --also none --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3 launches', d['gpu_launches'], d['steps'])"
