#!/bin/bash
# Bench every BASELINE config on one GPU (one JSON line each) + the reference
# arm on config 3 (the metric's configuration, the default).  Outputs
# gpurun_out/bench_cfg<N>.json, bench_ref_cfg3.json.
mkdir -p gpurun_out
for c in 3 1 0 2 4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_cfg$c.log 2>&1
  echo "cfg$c rc=$?"; tail -1 gpurun_out/bench_cfg$c.log > gpurun_out/bench_cfg$c.json
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_cfg3.log 2>&1
echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_cfg3.log > gpurun_out/bench_ref_cfg3.json
