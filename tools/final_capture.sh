# Evidence capture for profiles/r02 (run under gpurun; one GPU).  Every command exits
# before the next starts; numbers taken under ncu are never bench values.
set -x
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
./tools/micro/l1_peak > $O/l1_peak.json 2> $O/l1_peak.err
./tools/micro/l1_pattern > $O/l1_pattern.json 2> $O/l1_pattern.err
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider -rf --durations=25 > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; tail -c 300 $O/bench_c3.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --force-dist --steps 50 --no-cpu-baseline > $O/bench_c3_forcedist.json 2> $O/bench_c3_forcedist.err
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python tools/bench_configs.py --out $O/configs.json > $O/configs.log 2>&1
timeout 600 python tools/prof_slices.py c3 > $O/spdhg_slices_tax.json 2> $O/prof_slices.err
timeout 600 python tools/prof_shard.py --config c3 > $O/shard_local_gates_c3.txt 2>&1
timeout 900 python tools/prof_shard.py --config c4 --locals 5,10,20,40 --iters 5 > $O/shard_local_gates_c4.txt 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_timed.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_timed.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|adj_kernel|pack_kernel|update_kernel" -s 4 -c 4 -o $O/prof_c3_pdhg -f python tools/prof_iter.py --config c3 --mode pdhg --iters 3 > $O/ncu_pdhg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|adj_kernel|pack_kernel|update_kernel" -s 40 -c 4 -o $O/prof_c3_spdhg -f python tools/prof_iter.py --config c3 --mode spdhg --iters 20 > $O/ncu_spdhg.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"fwd_kernel|adj_kernel|pack_kernel|update_kernel" -s 4 -c 4 -o $O/prof_c4_pdhg -f python tools/prof_iter.py --config c4 --mode pdhg --iters 2 > $O/ncu_c4.log 2>&1
ls -la $O
