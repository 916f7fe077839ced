"""Per-CUDA-source-line totals from `ncu --page source --csv --print-source cuda,sass`:
instructions executed and stall samples, hottest lines first."""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
res, fname = [], None
h = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        ie = h.index("Instructions Executed")
        st = h.index("Warp Stall Sampling (All Samples)")
        continue
    if h is None or not r or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        res.append((fname, int(r[0]), r[1].strip()[:70], int(r[ie] or 0), int(r[st] or 0)))
    except (ValueError, IndexError):
        pass
te = sum(x[3] for x in res) or 1
ts = sum(x[4] for x in res) or 1
res.sort(key=lambda x: -x[3])
for f, ln, src, e, s in res[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{e / te * 100:5.1f}% ins {s / ts * 100:5.1f}% stall  {f}:{ln:<4d} {src}")
