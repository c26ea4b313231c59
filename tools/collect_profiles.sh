#!/bin/bash
# Turn a tools/final_capture.sh run (gpurun_out/r02) into the tracked profiles/r02 summaries.
set -e
O=${1:-gpurun_out/r02}; P=${2:-profiles/r02}
mkdir -p $P
for k in c3_pdhg c3_spdhg c4_pdhg; do
  python tools/ncu_summary.py $O/prof_$k.ncu-rep > $P/ncu_full_${k}_iteration.txt
done
python - "$O" <<'PY'
import ast, json, subprocess, sys
out = subprocess.run([sys.executable, "tools/ncu_traffic.py", sys.argv[1] + "/prof_c3_pdhg.ncu-rep"],
                     capture_output=True, text=True, check=True).stdout
json.dump(ast.literal_eval(out.strip().splitlines()[-1]), open("profiles/ncu_traffic.json", "w"), indent=1)
PY
python tools/launch_summary.py $O/launches_timed.csv > $P/launches_timed_region_summary.txt
cp $O/launches_timed.csv $P/launches_timed_region.csv
cp $O/bench_c3.json $P/bench_c3_n1.json
cp $O/bench_ref.json $P/bench_reference_arm.json
cp $O/bench_c3_forcedist.json $P/bench_c3_forcedist.json
cp $O/bench_c4.json $P/bench_c4_n1.json
cp $O/bench_c5.json $P/bench_c5_n1.json
cp $O/configs.json $O/configs.log $O/spdhg_slices_tax.json $O/shard_local_gates_c3.txt $O/shard_local_gates_c4.txt $P/
cp $O/l1_peak.json $O/l1_pattern.json profiles/
grep "PARITY" $O/pytest_gpu.log | sed 's/^\.*//' > $P/parity.txt
(grep -E "passed|failed" $O/pytest_gpu.log; grep -A26 "slowest 25" $O/pytest_gpu.log) > $P/pytest_gpu_summary.txt
python tools/sass_summary.py > $P/sass_summary.txt 2>/dev/null || true
