#!/bin/bash
# Bench every BASELINE config on one GPU (one JSON line each) + the reference
# arm on config 1.  Outputs gpurun_out/bench_cfg<N>.json, bench_ref_cfg1.json.
mkdir -p gpurun_out
for c in 1 0 2 4 3; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_cfg$c.log 2>&1
  echo "cfg$c rc=$?"; tail -1 gpurun_out/bench_cfg$c.log > gpurun_out/bench_cfg$c.json
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_cfg1.log 2>&1
echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_cfg1.log > gpurun_out/bench_ref_cfg1.json
