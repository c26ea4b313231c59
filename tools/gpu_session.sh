# GPU session script (run under gpurun)
timeout 900 python -m pytest tests/test_gpu_operators.py tests/test_gpu_solver.py -q -x -p no:cacheprovider -k "group or batch or large" > gpurun_out/gputest_grp.log 2>&1; echo rc=$? >> gpurun_out/gputest_grp.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_grp.log 2>&1; echo rc=$? >> gpurun_out/bench_grp.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_grp_c4.log 2>&1
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_grp_c5.log 2>&1
