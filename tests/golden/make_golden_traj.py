"""Golden outputs of the reference's ceiling inflation (trajectory.py:277-317)
on ceiling layers from the golden tomograms plus hand-made edge layers.
Build container only (imports tomoplan from /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_traj.py

Records sha256 of the float64 (flat, skirted) arrays per (layer, params).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent))

from tomoplan import trajectory  # noqa: E402  (reference, build container only)

import traj_cases  # noqa: E402

def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = dict(generator="tests/golden/make_golden_traj.py", reference="tomoplan 0.1.0",
               function="tomoplan.trajectory._inflate_ceiling", cases=[])
    for name, values, res in traj_cases.layers():
        for erosion, slope in traj_cases.PARAMS:
            flat, skirt = trajectory._inflate_ceiling(values, np.isfinite(values), res,
                                                      erosion, slope)
            out["cases"].append(dict(layer=name, res=res, erosion=erosion, slope=slope,
                                     values_sha256=sha(values), flat_sha256=sha(flat),
                                     skirted_sha256=sha(skirt)))
    (HERE / "golden_traj.json").write_text(json.dumps(out, indent=1))
    print(len(out["cases"]), "cases")


if __name__ == "__main__":
    main()
