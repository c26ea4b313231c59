#!/bin/bash
for defs in "$@"; do
  MCT_NVCC_EXTRA="$defs" python paper_2410_10503_b200/build.py --force > /dev/null 2>&1 || { echo "$defs BUILD FAILED"; continue; }
  for c in c3 c2 c1; do python tools/prof_spdhg.py --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$defs', d['config'], round(d['graph_epoch_ms'],4), {k: round(v,4) for k,v in d['kernel_ms_median'].items()})"; done
done
