#!/bin/bash
# A/B timing of libpct variants at one config: scripts/ab.sh <config> <lib1> <lib2> ...
# (alternating, 2 rounds; prints ms/map and stage times per run)
cfg=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    out=$(PCT_LIB=$lib timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu --no-parity 2>&1 | tail -1)
    python - "$lib" "$out" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[2]); s = d["stages_ms"]
    print(f"{sys.argv[1]:40s} {d['ms_per_step']:.3f} ms  " + " ".join(f"{k}={v:.3f}" for k, v in s.items()))
except Exception as e:
    print(sys.argv[1], "FAILED", sys.argv[2][-300:])
PY
  done
done
