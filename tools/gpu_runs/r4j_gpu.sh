# final check of the committed state: GPU suite, smoke, default bench line
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r4j_bench.json 2> gpurun_out/r4j_bench.err; tail -1 gpurun_out/r4j_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r4j_bench.json').read().strip().splitlines()[-1]); a=d['also']['C3']
print('C2', round(d['value'],1), round(d['ms_per_step']*1e3,1), d['gpu_launches'], round(d['roofline']['frac'],3), d['e2e']['value'], d['clocks'], '| C3', round(a['value'],1), a['gpu_launches'])"
