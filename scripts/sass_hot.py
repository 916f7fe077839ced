"""Summarise an `ncu --page source --csv` SASS listing: instructions executed
and stall samples per contiguous region, hottest first."""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ai, si, ie, sm = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ins = []
for r in rows[2:]:
    try:
        ins.append((r[ai], r[si], int(r[ie] or 0), int(r[sm] or 0)))
    except (ValueError, IndexError):
        pass
tot_e = sum(x[2] for x in ins); tot_s = sum(x[3] for x in ins)
print("total executed", tot_e, "samples", tot_s)
regs = []
cur = None
for a, s, e, st in ins:
    if cur and cur["e"] == e:
        cur["n"] += 1; cur["s"] += st; cur["ops"].append(s.split()[0] if s else "")
    else:
        cur = {"a": a, "e": e, "n": 1, "s": st, "ops": [s.split()[0] if s else ""]}
        regs.append(cur)
regs.sort(key=lambda r: -(r["e"] * r["n"]))
for r in regs[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    ops = {}
    for o in r["ops"]:
        ops[o] = ops.get(o, 0) + 1
    top = " ".join(f"{k}x{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:8])
    print(f"{r['a']:>6} n={r['n']:4d} exec={r['e']:9d} total={r['e']*r['n']/tot_e*100:5.1f}% stall={r['s']/max(1,tot_s)*100:5.1f}%  {top}")
