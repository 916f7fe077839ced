"""bench.py host helpers on CPU: the streamed archive checksum equals the
reference bench's checksum of the LGA bytes (tomoplan/bench.py:58-62), the
--gpus / WORLD_SIZE guard, and the reference arm on a small config."""

import hashlib
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

import oracle
from golden_util import TABLE_PARAMS
from oracle.archive import lga_bytes

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_streamed_checksum_equals_archive_checksum():
    from paper_2403_07631_b200 import synth
    xyz = synth.two_storey(30_000, seed=2)
    t = oracle.build(xyz, 0.5, 0.1)
    cost = oracle.evaluate(t["ground"], t["ceiling"], 0.1, TABLE_PARAMS)
    keep = oracle.simplify(t["ground"], cost)
    args = (t["heights"][keep], t["origin"], 0.1, t["z_min"], 0.5)
    want = hashlib.sha256(lga_bytes(t["ground"][keep], t["ceiling"][keep], cost[keep],
                                    *args)).hexdigest()[:16]
    got = bench.lga_sha256([t["ground"][k] for k in keep], [t["ceiling"][k] for k in keep],
                           [cost[k] for k in keep], [t["heights"][k] for k in keep],
                           t["origin"], 0.1, t["z_min"], 0.5)
    assert got == want


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_reference_arm_line():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config",
                        "0", "--steps", "1", "--warmup", "0"], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "Mpts/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert line["config"]["workload"].startswith("cfg0 two_storey")
