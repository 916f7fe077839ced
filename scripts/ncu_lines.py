"""CUDA source lines of one kernel carrying the most warp-stall samples and
instructions (ncu --page source --print-source cuda,sass).

    python scripts/ncu_lines.py report.ncu-rep <ncu-kernel-regex> [n]
"""
import csv
import subprocess
import sys


def main(rep, kre, n=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    path, hdr, agg = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
        elif r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0] not in ("",):
            st = int(r[4] or 0)
            ie = int(r[7] or 0)
            agg.append((st, ie, f"{path}:{r[0]}", r[1].strip()[:80]))
    tot = max(1, sum(a[0] for a in agg))
    itot = max(1, sum(a[1] for a in agg))
    print("stall samples", tot, "warp instructions", itot)
    for st, ie, loc, src in sorted(agg, reverse=True)[:n]:
        print(f"{100 * st / tot:5.1f}% stalls {100 * ie / itot:5.1f}% instr  {loc:28s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
