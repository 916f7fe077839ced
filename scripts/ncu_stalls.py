"""Instructions carrying the most warp-stall samples of one kernel in an ncu report.

    python scripts/ncu_stalls.py report.ncu-rep <ncu-kernel-regex> <name-substring> [min_pct]
"""
import csv
import subprocess
import sys


def main(rep, kre, sub, min_pct=0.6):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            secs.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
            cur["rows"].append(r)
    sec = [s for s in secs if sub in s["name"]][0]
    h = sec["hdr"]
    ie, src, st = h.index("Instructions Executed"), h.index("Source"), \
        h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ie] or 0) for r in sec["rows"])
    stot = max(1, sum(int(r[st] or 0) for r in sec["rows"]))
    print(sec["name"][:110])
    print("warp instructions", tot, "stall samples", stot)
    for r in sec["rows"]:
        v, s = int(r[ie] or 0), int(r[st] or 0)
        if 100 * s / stot >= min_pct:
            print(f"{r[0]:>6} {v:>11} {100 * s / stot:5.1f}%  {r[src].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else 0.6)
