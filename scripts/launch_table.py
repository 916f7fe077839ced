"""Per-kernel device times from an ncu --csv launch list (gpurun_out/launches_<tag>.csv):
the second half of the launches (the timed step after the warm-up step)."""
import collections, csv, sys
from pathlib import Path

for tag in sys.argv[1:]:
    rows = [r for r in csv.reader(l for l in Path(f"gpurun_out/launches_{tag}.csv").read_text().splitlines()
                                  if not l.startswith("=="))]
    h = rows[0]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        per.setdefault(r[ii], {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    launches = list(per.values())
    half = [v for v in launches[len(launches) // 2:]
            if "pct::" in v["kernel"] or "unnamed>::" in v["kernel"]]
    tot = sum(v.get("gpu__time_duration.sum", 0) for v in half)
    print(f"== {tag}: {len(half)} launches, {tot / 1e3:.1f} us")
    for v in half:
        t = v.get("gpu__time_duration.sum", 0)
        rd = v.get("dram__bytes_read.sum", 0) / 1e6
        wr = v.get("dram__bytes_write.sum", 0) / 1e6
        print(f"  {t / 1e3:8.1f} us  {rd:8.1f} MB rd {wr:8.1f} MB wr  {v['kernel'][:90]}")
