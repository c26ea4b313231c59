# GPU session script (run under gpurun)
mkdir -p gpurun_out/s1
timeout 900 python -m pytest tests/test_gpu_chunked.py -q -x -p no:cacheprovider > gpurun_out/s1/chunked.log 2>&1; echo rc=$? >> gpurun_out/s1/chunked.log
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_chunked.py > gpurun_out/s1/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/s1/gpu_all.log
timeout 300 python tools/mem_breakdown.py c3 c4 > gpurun_out/s1/mem.json 2> gpurun_out/s1/mem.err
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/s1/bench_c3.json 2> gpurun_out/s1/bench_c3.err
timeout 600 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s1/bench_c4.json 2> gpurun_out/s1/bench_c4.err
timeout 600 python bench.py --config c5 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/s1/bench_c5.json 2> gpurun_out/s1/bench_c5.err
