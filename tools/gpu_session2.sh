# K2 lane-interleave sweep (run under gpurun)
mkdir -p gpurun_out/s2
bash tools/sweep_build.sh "-DMCT_FWD_IL=4" "-DMCT_FWD_IL=4 -DMCT_FWD_ANGLES=2 -DFWD_MIN_BLOCKS2=16" "-DMCT_FWD_IL=4 -DMCT_FWD_ANGLES=2 -DFWD_MIN_BLOCKS2=14" "-DMCT_FWD_IL=1" > gpurun_out/s2/sweep_il.txt 2>&1
python paper_2410_10503_b200/build.py --force > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_chunked.py -q -p no:cacheprovider > gpurun_out/s2/chunked.log 2>&1
