#!/bin/bash
# K2 (gate pairs) occupancy / block-shape / lane-interleave sweep on the C3 PDHG epoch
# (run under gpurun; DESIGN.md §9 holds the round-2 results).  Rebuilds the default at the end.
mkdir -p gpurun_out/sweep
bash tools/sweep_build.sh "-DFWD_MIN_BLOCKS2=8" "-DFWD_MIN_BLOCKS2=9" "-DFWD_MIN_BLOCKS2=10" "-DFWD_MIN_BLOCKS2=12" \
  "-DMCT_FWD_ANGLES=8 -DFWD_MIN_BLOCKS2=4" "-DMCT_FWD_ANGLES=8 -DFWD_MIN_BLOCKS2=5" \
  "-DMCT_FWD_ANGLES=2 -DFWD_MIN_BLOCKS2=16" "-DMCT_FWD_ANGLES=2 -DFWD_MIN_BLOCKS2=20" \
  "-DFWD_CARVEOUT_PCT=0" "-DFWD_CARVEOUT_PCT=15" \
  "-DMCT_FWD_IL=4" "-DMCT_FWD_IL=4 -DMCT_FWD_ANGLES=2 -DFWD_MIN_BLOCKS2=16" "-DMCT_FWD_IL=1" \
  > gpurun_out/sweep/k2_shapes.txt 2>&1
python paper_2410_10503_b200/build.py --force > /dev/null 2>&1
