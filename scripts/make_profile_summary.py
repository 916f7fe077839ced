"""Copy the ncu evidence of one gpurun call into profiles/ (tracked).

    python scripts/make_profile_summary.py <tag> <round-name> [config]

Writes profiles/<round>_launches.csv (per-launch device time + DRAM bytes of one
bench step, from `ncu --metrics gpu__time_duration.sum,dram__bytes_*`),
profiles/<round>_<kernel>_ncu.txt (the --set full details page of the top
kernel + its SASS opcode histogram) and updates profiles/ncu_traffic.json
(DRAM bytes per launch of the evaluate kernel, read by bench.py)."""
import collections, csv, io, json, re, subprocess, sys
from pathlib import Path

tag, rnd = sys.argv[1], sys.argv[2]
cfg = sys.argv[3] if len(sys.argv) > 3 else "cfg1"
out = Path("profiles"); out.mkdir(exist_ok=True)
src = Path(f"gpurun_out/launches_{tag}.csv")
rows = [r for r in csv.reader(l for l in src.read_text().splitlines() if not l.startswith("=="))]
h = rows[0]; ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.OrderedDict()
for r in rows[1:]:
    per.setdefault(r[ii], {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
launches = list(per.values())
half = launches[len(launches) // 2:]  # the timed step (after the warm-up step)
# the library's kernels (the L2 flush between steps is not in the step)
half = [v for v in half if "pct::" in v["kernel"] or "unnamed>::" in v["kernel"]]
tot = sum(v.get("gpu__time_duration.sum", 0) for v in half)
with open(out / f"{rnd}_launches.csv", "w") as f:
    f.write("kernel,time_us,share,dram_read_MB,dram_write_MB\n")
    for v in half:
        t = v.get("gpu__time_duration.sum", 0)
        f.write(f"\"{v['kernel'][:90]}\",{t/1e3:.1f},{t/tot:.3f},"
                f"{v.get('dram__bytes_read.sum',0)/1e6:.1f},{v.get('dram__bytes_write.sum',0)/1e6:.1f}\n")
rep = Path(sys.argv[4]) if len(sys.argv) > 4 else Path(f"gpurun_out/prof_{tag}.ncu-rep")
if rep.exists():
    # one details page (+ SASS opcode histogram) per kernel in the report
    det = subprocess.run(["ncu", "-i", str(rep), "--page", "details", "--csv"], capture_output=True, text=True).stdout
    lines = list(csv.reader(io.StringIO(det)))
    hh = lines[0]
    si, mi2, vi2, ui, ki2, ii2 = (hh.index(x) for x in ("Section Name", "Metric Name", "Metric Value",
                                                         "Metric Unit", "Kernel Name", "ID"))
    by = collections.OrderedDict()
    for r in lines[1:]:
        by.setdefault(r[ii2], []).append(r)
    seen = collections.Counter()
    for rid, rs in by.items():
        kname = rs[0][ki2]
        short = re.sub(r"[^a-z_]", "", kname.split("(")[0].split("::")[-1].split("<")[0])
        seen[short] += 1
        if seen[short] > 1:  # another instantiation of the same kernel
            short = f"{short}{seen[short]}"
        body = [f"ncu --set full --clock-control none --import-source on, report {rep.name}, launch id {rid}",
                f"kernel: {kname}", ""]
        for r in rs:
            body.append(f"{r[si][:30]:30s} {r[mi2][:55]:55s} {r[vi2]} {r[ui]}")
        ops = subprocess.run([sys.executable, "scripts/ncu_ops.py", str(rep), "24", short],
                             capture_output=True, text=True).stdout
        (out / f"{rnd}_{short}_ncu.txt").write_text("\n".join(body) + "\n\nSASS opcode histogram:\n" + ops)
tr_path = out / "ncu_traffic.json"
tr = json.loads(tr_path.read_text()) if tr_path.exists() else {}
# the evaluate stage = every launch between the build scan and the simplify window
ev = [v for v in half if any(x in v["kernel"] for x in ("eval", "terrain_walk", "resolve_inflate",
                                                          "zero_pads", "change_mask"))]
if ev:
    tr[cfg] = {"kernels": sorted({v["kernel"][:80] for v in ev}),
               "eval_dram_bytes": sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in ev),
               "eval_time_us_ncu": sum(v.get("gpu__time_duration.sum", 0) for v in ev) / 1e3,
               "source": f"{rnd}_launches.csv"}
tr_path.write_text(json.dumps(tr, indent=1))
print("wrote", sorted(p.name for p in out.iterdir()))
