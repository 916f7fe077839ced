"""Golden outcomes of the reference's binary PCD loader (cloud_io.py:123-168)
on the files of tests/pcd_cases.py.  Build container only (imports tomoplan
from /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_pcd.py

For every case records either the loaded cloud (point count, dropped rows,
sha256 of the float64 (N, 3) xyz bytes, sha256 of the file itself) or the
exception type and message (the file path replaced by "<path>").
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent))

from tomoplan import cloud_io  # noqa: E402  (reference, build container only)

import pcd_cases  # noqa: E402


def main():
    out = dict(generator="tests/golden/make_golden_pcd.py", reference="tomoplan 0.1.0",
               loader="tomoplan.cloud_io.load_cloud(path, 'pcd_binary')", cases={})
    with tempfile.TemporaryDirectory() as d:
        for name in pcd_cases.CASES:
            path = pcd_cases.write_case(name, d)
            rec = dict(file_sha256=hashlib.sha256(path.read_bytes()).hexdigest())
            try:
                cloud = cloud_io.load_cloud(path, "pcd_binary")
            except Exception as exc:  # noqa: BLE001 — the outcome is the record
                rec.update(error=type(exc).__name__, message=str(exc).replace(str(path), "<path>"))
            else:
                xyz = np.ascontiguousarray(cloud.xyz)
                assert xyz.dtype == np.float64
                rec.update(n=int(xyz.shape[0]), dropped=int(cloud.dropped),
                           xyz_sha256=hashlib.sha256(xyz.tobytes()).hexdigest())
            out["cases"][name] = rec
            print(name, {k: v for k, v in rec.items() if k != "file_sha256"})
    (HERE / "golden_pcd.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
