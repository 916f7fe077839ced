"""Print the bench line, the launch list and the top-kernel ncu numbers from gpurun_out/."""
import csv, json, sys, subprocess, collections, re
tag = sys.argv[1] if len(sys.argv) > 1 else "cur"
try:
    print(open("gpurun_out/pytest_gpu.log").read().strip().splitlines()[-1])
except Exception as e:
    print("no pytest log", e)
try:
    d = json.loads(open("gpurun_out/bench.log").readline())
    print("value %.1f Mpts/s  ms/step %.4f" % (d["value"], d["ms_per_step"]), {k: round(v, 4) for k, v in d["stages_ms"].items()})
    r = d["roofline"]; print("eval roofline %.0f GB/s frac %.3f" % (r["achieved"], r["frac"]), "clocks", d["clocks"])
    if "e2e" in d: print("e2e ms %.3f value %.1f" % (d["e2e"]["ms_per_step"], d["e2e"]["value"]))
    if "cpu_baseline" in d: print("cpu", d["cpu_baseline"]["value"], d["cpu_baseline"]["cores"])
except Exception as e:
    print("no bench", e)
rows = [r for r in csv.reader(l for l in open(f"gpurun_out/launches_{tag}.csv") if not l.startswith("=="))]
h = rows[0]; ki = h.index("Kernel Name"); mi = h.index("Metric Name"); vi = h.index("Metric Value"); ii = h.index("ID")
per = collections.OrderedDict()
for r in rows[1:]:
    per.setdefault(r[ii], {"k": r[ki][:50]})[r[mi]] = float(r[vi].replace(",", ""))
for v in list(per.values())[len(per)//2:]:
    print(f"  {v['k']:50s} {v.get('gpu__time_duration.sum',0)/1e3:9.1f} us  rd {v.get('dram__bytes_read.sum',0)/1e6:8.1f} MB  wr {v.get('dram__bytes_write.sum',0)/1e6:8.1f} MB")
