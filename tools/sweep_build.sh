#!/bin/bash
# tuning sweep: rebuild with -D overrides and time the C3 PDHG / SPDHG epochs
for defs in "$@"; do
  MCT_NVCC_EXTRA="$defs" python paper_2410_10503_b200/build.py --force > /dev/null 2>&1 || { echo "$defs BUILD FAILED"; continue; }
  python bench.py --no-cpu-baseline --no-e2e --steps 50 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$defs', round(d['value'],1), {k: round(v,3) for k,v in d['kernel_ms'].items()}, round(d['spdhg']['value'],1))"
done
