#!/bin/bash
# GPU-box check used during development: GPU tests (summary line), then one bench line summary.
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -x -q 2>&1 | grep -E "FAILED|Error|passed|failed" | head -5
python bench.py --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
k = d['kernels_ms']
print('value %.2f Gcells/s  step %.4f ms  e2e %.4f ms  | prologue %.1f  pass1 %.1f  pass2a %.1f  2b %.1f  epi %.1f us  | launches %d  roof %.2f' % (
    d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], 1e3 * k['maxv_ms'], 1e3 * k['weights_scan_ms'],
    1e3 * k['bin_reduce_ms'], 1e3 * k.get('bin_boundary_ms', 0), 1e3 * k['epilogue_ms'], d['gpu_launches'], d['roofline']['frac']))"
