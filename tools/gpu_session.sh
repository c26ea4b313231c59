# GPU session script (run under gpurun)
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest3.log 2>&1; echo rc=$? >> gpurun_out/gputest3.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench3.log 2>&1; echo rc=$? >> gpurun_out/bench3.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3_c4.log 2>&1
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3_c5.log 2>&1
