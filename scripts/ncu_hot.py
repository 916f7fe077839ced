"""Hot SASS blocks of one kernel in an ncu report (source page, SASS view).

    python scripts/ncu_hot.py report.ncu-rep <kernel-regex> [n_blocks]
"""
import csv
import subprocess
import sys


def main(rep, kern, nb=8):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    sections, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            sections.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
            cur["rows"].append(r)
    import re
    sec = next(s for s in sections if re.search(kern, s["name"]))
    h = sec["hdr"]
    ie, src, st = h.index("Instructions Executed"), h.index("Source"), \
        h.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[ie] or 0), int(r[st] or 0), r[src].strip()) for r in sec["rows"]]
    tot = sum(d[0] for d in data)
    stot = max(1, sum(d[1] for d in data))
    print(sec["name"][:120])
    print("total warp instructions", tot, "stall samples", stot)
    blocks, cur = [], None
    for i, (v, s, t) in enumerate(data):
        if cur and v == cur[0]:
            cur[2] += 1
            cur[3] += s
            cur[4].append(t)
        else:
            cur = [v, i, 1, s, [t]]
            blocks.append(cur)
    blocks.sort(key=lambda b: -b[0] * b[2])
    for b in blocks[:nb]:
        print(f"x{b[0]} len {b[2]} = {100 * b[0] * b[2] / tot:.1f}% of instr, "
              f"{100 * b[3] / stot:.1f}% of stalls:")
        for t in b[4][:48]:
            print("     ", t[:96])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 8)
