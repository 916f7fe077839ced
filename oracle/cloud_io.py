"""Oracle: binary PCD payload -> (N, 3) float64 points + dropped count.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  A numpy restatement of the
reference's binary branch of ``_load_pcd`` (tomoplan/cloud_io.py:123-146) and
``_keep_finite`` (:53-55): the payload is viewed as little-endian records,
x/y/z are taken from their byte offsets, up-cast to float64 and the rows with
a non-finite coordinate removed, order kept.  Header parsing is shared with
the product (``paper_2403_07631_b200.cloud_io.read_pcd_header`` is host logic,
not computation); the payload arithmetic here is independent of the device
path it checks.  Pinned by tests/golden/golden_pcd.json (reference outcomes).
"""

from __future__ import annotations

import numpy as np


def extract(payload: bytes, n_records: int, record_bytes: int, offsets) -> tuple[np.ndarray, int]:
    """x/y/z float32 at byte ``offsets`` of ``n_records`` records ->
    (finite rows as float64 (M, 3), number of dropped rows)."""
    raw = np.frombuffer(payload, np.uint8, count=n_records * record_bytes)
    raw = raw.reshape(n_records, record_bytes)
    cols = [raw[:, o:o + 4].copy().view("<f4").reshape(n_records) for o in offsets]
    pts = np.stack(cols, axis=1).astype(np.float64)          # cloud_io.py:146
    good = np.isfinite(pts).all(axis=1)                      # cloud_io.py:54
    return pts[good], int(n_records - good.sum())            # cloud_io.py:55
