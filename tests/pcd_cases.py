"""Deterministic binary-PCD test files (layouts, non-finite rows, malformed
headers) shared by tests/golden/make_golden_pcd.py (which records what the
reference's loader, cloud_io.py:123-168, returns for each) and the tests.

Each case is a function writing one file; the payloads come from a seeded
PCG64 generator, so the files are byte-identical wherever they are made.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

_NP = {"F": "f", "I": "i", "U": "u"}


def _header(fields, n, data="binary", extra=(), lowercase=False, comments=False,
            points=None, omit=()):
    names = " ".join(f[0] for f in fields)
    lines = []
    if comments:
        lines += ["# .PCD v0.7 - test file", "", "   # indented comment"]
    rows = [("VERSION", "0.7"), ("FIELDS", names),
            ("SIZE", " ".join(str(f[1]) for f in fields)),
            ("TYPE", " ".join(f[2] for f in fields)),
            ("COUNT", " ".join(str(f[3]) for f in fields)),
            ("WIDTH", str(n)), ("HEIGHT", "1"), ("VIEWPOINT", "0 0 0 1 0 0 0"),
            ("POINTS", str(n) if points is None else points), ("DATA", data)]
    for key, val in rows:
        if key in omit:
            continue
        lines.append(f"{key.lower() if lowercase else key} {val}")
    lines += list(extra)
    return ("\n".join(lines) + "\n").encode("ascii")


def _records(fields, n, seed, nonfinite=0.0, all_nonfinite=False):
    dt = np.dtype([(f[0], f"<{_NP[f[2]]}{f[1]}", (f[3],)) if f[3] > 1
                   else (f[0], f"<{_NP[f[2]]}{f[1]}") for f in fields])
    rng = np.random.default_rng(seed)
    rec = np.zeros(n, dt)
    for name in dt.names:
        sub = rec[name]
        if sub.dtype.kind == "f":
            rec[name] = rng.uniform(-50.0, 50.0, sub.shape).astype(sub.dtype)
        else:
            info = np.iinfo(sub.dtype)
            rec[name] = rng.integers(0, min(info.max, 1 << 20), sub.shape, endpoint=False)
    if nonfinite or all_nonfinite:
        bad = np.ones(n, bool) if all_nonfinite else rng.random(n) < nonfinite
        which = rng.integers(0, 3, n)
        vals = np.array([np.nan, np.inf, -np.inf], np.float32)[rng.integers(0, 3, n)]
        for k, axis in enumerate("xyz"):
            m = bad & (which == k)
            rec[axis][m] = vals[m]
        if all_nonfinite:
            rec["x"][:] = np.nan
        # NaN in a non-coordinate field does not drop the row
        for name in dt.names:
            if name not in "xyz" and rec[name].dtype.kind == "f":
                rec[name][rng.random(n) < 0.2] = np.nan
    return rec


XYZ = [("x", 4, "F", 1), ("y", 4, "F", 1), ("z", 4, "F", 1)]


def _spec(fields, n, seed, **kw):
    return dict(fields=fields, n=n, seed=seed, **kw)


CASES = {
    "plain_xyz": _spec(XYZ, 5000, 1),
    "xyz_intensity": _spec(XYZ + [("intensity", 4, "F", 1)], 7001, 2),
    "mixed_counts": _spec([("rgb", 4, "U", 1), ("x", 4, "F", 1), ("normal", 4, "F", 3),
                           ("y", 4, "F", 1), ("ring", 2, "U", 1), ("z", 4, "F", 1)], 4099, 3),
    "unaligned_u1": _spec([("label", 1, "U", 1), ("x", 4, "F", 1), ("y", 4, "F", 1),
                           ("z", 4, "F", 1), ("t", 8, "F", 1), ("flag", 1, "I", 1)], 3001, 4),
    "reordered": _spec([("z", 4, "F", 1), ("t", 8, "F", 1), ("y", 4, "F", 1),
                        ("x", 4, "F", 1)], 2500, 5),
    "nonfinite_rows": _spec(XYZ + [("intensity", 4, "F", 1)], 20000, 6, nonfinite=0.03),
    "comments_lowercase": _spec(XYZ, 1500, 7, lowercase=True, comments=True),
    "trailing_bytes": _spec(XYZ, 1000, 8, trailing=37),
    "no_count_line": _spec(XYZ + [("i", 2, "I", 1)], 1200, 9, omit=("COUNT",)),
    "multi_tile": _spec(XYZ + [("intensity", 4, "F", 1)], 300_001, 10, nonfinite=0.001),
    # errors
    "all_nonfinite": _spec(XYZ, 800, 11, all_nonfinite=True),
    "zero_points": _spec(XYZ, 0, 12),
    "truncated": _spec(XYZ, 1000, 13, truncate=5),
    "ascii_data": _spec(XYZ, 10, 14, data="ascii"),
    "compressed_data": _spec(XYZ, 10, 15, data="binary_compressed"),
    "x_float64": _spec([("x", 8, "F", 1), ("y", 4, "F", 1), ("z", 4, "F", 1)], 10, 16),
    "x_count2": _spec([("x", 4, "F", 2), ("y", 4, "F", 1), ("z", 4, "F", 1)], 10, 17),
    "bad_type": _spec(XYZ + [("q", 4, "X", 1)], 10, 18),
    "missing_z": _spec([("x", 4, "F", 1), ("y", 4, "F", 1)], 10, 19),
    "no_data_line": _spec(XYZ, 10, 20, omit=("DATA",)),
    "bad_points": _spec(XYZ, 10, 21, points="many"),
    "no_fields": _spec(XYZ, 10, 22, omit=("FIELDS",)),
}


def write_case(name: str, directory) -> Path:
    """Write case `name` as <directory>/<name>.pcd and return the path."""
    c = CASES[name]
    path = Path(directory) / f"{name}.pcd"
    fields, n = c["fields"], c["n"]
    head = _header(fields, n, data=c.get("data", "binary"), lowercase=c.get("lowercase", False),
                   comments=c.get("comments", False), points=c.get("points"),
                   omit=c.get("omit", ()))
    ok_types = all(f[2] in _NP for f in fields)
    payload = b""
    if ok_types:
        rec = _records(fields, n, c["seed"], c.get("nonfinite", 0.0),
                       c.get("all_nonfinite", False))
        payload = rec.tobytes()
    else:
        payload = np.random.default_rng(c["seed"]).bytes(n * sum(f[1] * f[3] for f in fields))
    if c.get("truncate"):
        payload = payload[:-c["truncate"]]
    payload += b"\x00" * c.get("trailing", 0)
    path.write_bytes(head + payload)
    return path
