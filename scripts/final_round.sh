#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, every bench line, ncu
# launch lists (cfg0-3) and --set full captures of the timed step's kernels
# (cfg3: the build / evaluate / simplify kernels; cfg1: the small-map ones).
mkdir -p gpurun_out; export PYTHONPATH=$PWD
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
bash scripts/bench_all.sh
PCT_XFER_TRACE=1 timeout 600 python scripts/e2e_split.py > gpurun_out/e2e_split.txt 2>&1; echo "e2e_split rc=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/red_peak scripts/red_peak.cu && /tmp/red_peak > gpurun_out/red_peak.json
for c in 0 1 2 3; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_f$c.csv \
    python bench.py --config $c --profile --no-e2e --no-cpu --no-parity > /dev/null 2>&1
  echo "ncu list cfg$c rc=$?"
done
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"hist_pass|hist_reduce|terrain_walk|resolve_inflate_bnb|window" -s 6 -c 6 \
  -o gpurun_out/prof_f3 python bench.py --config 3 --profile --no-e2e --no-cpu --no-parity > gpurun_out/ncu_full3.log 2>&1
echo "ncu full cfg3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"terrain_walk|resolve_inflate_bnb|scatter_kernel|scan_kernel|window_kernel" -s 5 -c 5 \
  -o gpurun_out/prof_f1 python bench.py --config 1 --profile --no-e2e --no-cpu --no-parity > gpurun_out/ncu_full1.log 2>&1
echo "ncu full cfg1 rc=$?"
