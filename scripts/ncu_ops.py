"""Opcode histogram + hottest basic blocks of one ncu report (SASS source page)."""
import csv, re, sys, subprocess, collections, io
rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3], "-c", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia = h.index("Source"); ie = h.index("Instructions Executed"); iw = h.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter(); st = collections.Counter(); tot = totw = 0
seq = []
for r in rows[2:]:
    if len(r) <= ie or not r[ie].isdigit(): continue
    src = r[ia].strip(); m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", src)
    if not m: continue
    op = m.group(2).split(".")[0]; n = int(r[ie] or 0); w = int(r[iw] or 0)
    ops[op] += n; st[op] += w; tot += n; totw += w; seq.append((src, n, w))
print("total warp instr", tot)
for op, n in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 16):
    print(f"  {op:10s} {n:11d} {100*n/tot:5.1f}%  stalls {100*st[op]/max(totw,1):5.1f}%")
blocks = []; cur = None
for i, (s, n, w) in enumerate(seq):
    if cur and cur[1] == n: cur[2].append(s); cur[3] += w
    else: cur = [i, n, [s], w]; blocks.append(cur)
for b in sorted(blocks, key=lambda b: -b[1] * len(b[2]))[:10]:
    print(f"block@{b[0]} x{b[1]} len {len(b[2])} {100*b[1]*len(b[2])/tot:.1f}% stalls {100*b[3]/max(totw,1):.1f}%: " + " | ".join(x[:28] for x in b[2][:8]))
