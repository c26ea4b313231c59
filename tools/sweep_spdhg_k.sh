#!/bin/bash
# tuning sweep of the single-gate SPDHG iteration: rebuild with -D overrides and
# print the per-kernel medians of tools/prof_spdhg.py
cfg=${CFG:-c3}
for defs in "$@"; do
  MCT_NVCC_EXTRA="$defs" python paper_2410_10503_b200/build.py --force > /dev/null 2>&1 || { echo "$defs BUILD FAILED"; continue; }
  python tools/prof_spdhg.py --config $cfg 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$defs', {k: round(v*1000,1) for k,v in d['kernel_ms_median'].items()}, 'graph_iter_us', round(d['graph_iter_ms']*1000,1))"
done
