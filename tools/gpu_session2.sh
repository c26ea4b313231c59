# K2 occupancy / block-shape sweep after the lane interleave (run under gpurun)
mkdir -p gpurun_out/s2
bash tools/sweep_build.sh "-DFWD_MIN_BLOCKS2=8" "-DFWD_MIN_BLOCKS2=9" "-DFWD_MIN_BLOCKS2=10" "-DFWD_MIN_BLOCKS2=12" \
  "-DMCT_FWD_ANGLES=8 -DFWD_MIN_BLOCKS2=4" "-DMCT_FWD_ANGLES=8 -DFWD_MIN_BLOCKS2=5" "-DMCT_FWD_ANGLES=2 -DFWD_MIN_BLOCKS2=16" "-DMCT_FWD_ANGLES=2 -DFWD_MIN_BLOCKS2=20" \
  "-DFWD_CARVEOUT_PCT=0" "-DFWD_CARVEOUT_PCT=15" > gpurun_out/s2/sweep_k2.txt 2>&1
python paper_2410_10503_b200/build.py --force > /dev/null 2>&1
