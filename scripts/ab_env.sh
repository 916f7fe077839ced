#!/bin/bash
# A/B timing of environment settings at one config:
#   scripts/ab_env.sh <config> "VAR=a" "VAR=b" ...   (alternating, 2 rounds)
cfg=$1; shift
for rep in 1 2; do
  for e in "$@"; do
    out=$(env $e timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu --no-parity 2>&1 | tail -1)
    python - "$e" "$out" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[2]); s = d["stages_ms"]
    print(f"{sys.argv[1]:40s} {d['ms_per_step']:.3f} ms  " + " ".join(f"{k}={v:.3f}" for k, v in s.items()))
except Exception as e:
    print(sys.argv[1], "FAILED", sys.argv[2][-300:])
PY
  done
done
