"""Summarise an ncu --set full report: key metrics per kernel launch.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [> profiles/..txt]
"""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Issue Slots Busy", "Executed Instructions",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Block Limit Registers", "Block Limit Shared Mem", "Waves Per SM", "Compute (SM) Throughput"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_requests_op_red.sum",
       "lts__t_requests_op_atom.sum", "smsp__inst_executed_op_shared_atom.sum",
       "l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum", "smsp__sass_inst_executed_op_global_red.sum",
       "smsp__sass_inst_executed_op_shared_atom.sum", "lts__t_sectors_op_red.sum",
       "gpu__time_duration.sum"]


def rows(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(out.splitlines()))


def main(rep):
    det = rows(rep, "details")
    h = det[0]
    per = {}
    for r in det[1:]:
        d = dict(zip(h, r))
        key = (d["ID"], d["Kernel Name"])
        per.setdefault(key, {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    raw = rows(rep, "raw")
    rh = raw[0]
    rawd = {}
    for r in raw[2:]:
        d = dict(zip(rh, r))
        rawd[(d.get("ID"), d.get("Kernel Name"))] = d
    for key, m in per.items():
        print(f"== launch {key[0]}: {key[1][:110]}")
        for k in KEYS:
            if k in m:
                print(f"   {k:38s} {m[k][0]} {m[k][1]}")
        rd = rawd.get(key, {})
        for k in RAW:
            if k in rd and rd[k] not in ("", "n/a"):
                print(f"   {k:38s} {rd[k]}")


if __name__ == "__main__":
    main(sys.argv[1])
