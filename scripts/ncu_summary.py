"""Summarise an ncu report (raw page) or a launch-list CSV into markdown for profiles/.

    python scripts/ncu_summary.py full  gpurun_out/x.ncu-rep  > profiles/...md
    python scripts/ncu_summary.py launches gpurun_out/launches.csv > profiles/...md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    print(f"# ncu --set full: `{rep.split('/')[-1]}`\n")
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        print(f"## {d.get('Kernel Name', '?')[:140]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS + sorted(k for k in head if "pipe_tensor" in k and "pct" in k and k not in KEYS):
            if k in d and d[k] != "":
                print(f"| {k} | {d[k]} | {u.get(k, '')} |")
        print()


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r.get("Metric Unit"), 1.0)
        name = r["Kernel Name"].split("(")[0].replace("void ", "")[:70]
        agg[name][0] += 1
        agg[name][1] += v * scale
        total += v * scale
    print(f"# ncu launch list: `{path.split('/')[-1]}` (cold-cache, serialised)\n")
    print(f"total {total / 1000:.3f} ms over {sum(a[0] for a in agg.values())} launches\n")
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n} | {t:.1f} | {100 * t / total:.1f}% |")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
