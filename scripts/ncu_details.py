"""Key ncu --set full metrics per kernel launch from a `--page details --csv`
export:  python scripts/ncu_details.py DETAILS.csv [kernel-regex]"""
import csv, re, sys
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy",
        "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block",
        "Block Limit Registers", "Block Limit Shared Mem", "Waves Per SM", "Mem Busy",
        "Max Bandwidth", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Branch Instructions Ratio", "Executed Instructions"]
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
I = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "Grid Size", "Block Size")}
out = {}
for r in rows[1:]:
    if len(r) < len(h) - 5:
        continue
    name = re.sub(r"\(.*", "", r[I["Kernel Name"]]).replace("unnamed>::", "")
    if pat and not pat.search(name):
        continue
    key = (int(r[I["ID"]]), name, r[I["Grid Size"]], r[I["Block Size"]])
    if r[I["Metric Name"]] in KEYS:
        out.setdefault(key, {})[r[I["Metric Name"]]] = r[I["Metric Value"]] + " " + r[I["Metric Unit"]]
for key, m in out.items():
    print(f"#{key[0]} {key[1]} grid {key[2]} block {key[3]}")
    for k in KEYS:
        if k in m:
            print(f"    {k:36s} {m[k]}")
