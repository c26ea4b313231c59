# Evidence capture for profiles/rNN (run under gpurun; one GPU)
set -x
./tools/micro/l1_peak > gpurun_out/l1_peak.json 2> gpurun_out/l1_peak.err
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 300 gpurun_out/bench_c3.json
timeout 600 python bench.py --impl reference --steps 40 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python tools/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_timed.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_timed.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|adj_kernel|pack_kernel|update_kernel" -s 4 -c 4 -o gpurun_out/prof_c3_pdhg_r02 -f python tools/prof_iter.py --config c3 --mode pdhg --iters 3 > gpurun_out/ncu_pdhg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|adj_kernel|pack_kernel|update_kernel" -s 40 -c 4 -o gpurun_out/prof_c3_spdhg_r02 -f python tools/prof_iter.py --config c3 --mode spdhg --iters 20 > gpurun_out/ncu_spdhg.log 2>&1
ls -la gpurun_out/
