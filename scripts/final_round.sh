#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, every bench line, ncu
# launch lists (cfg1-3) and --set full captures of the timed step's kernels.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
bash scripts/bench_all.sh
for c in 1 2 3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_f$c.csv \
    python bench.py --config $c --profile --no-e2e --no-cpu > /dev/null 2>&1
  echo "ncu list cfg$c rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"terrain_walk|resolve_inflate_bnb|scatter_kernel|scan_kernel|window_kernel" -s 5 -c 5 \
  -o gpurun_out/prof_f1 python bench.py --profile --no-e2e --no-cpu > gpurun_out/ncu_full1.log 2>&1
echo "ncu full cfg1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"terrain_walk|resolve_inflate_bnb" -s 2 -c 2 \
  -o gpurun_out/prof_f2 python bench.py --config 2 --profile --no-e2e --no-cpu > gpurun_out/ncu_full2.log 2>&1
echo "ncu full cfg2 rc=$?"
