"""DRAM traffic per bench step, per library stage, from an ncu --set full
capture of `bench.py --steps S --warmup W --no-secondary --no-cpu-baseline`:

    python scripts/ncu_traffic.py REPORT STEPS_CAPTURED OUT.json

STEPS_CAPTURED = the number of complete layer steps inside the capture (warm-up
+ timed + e2e steps); the kernels' dram__bytes_read.sum + dram__bytes_write.sum
are summed per library stage name and divided by it (ncu replays each kernel
with a cold cache, so these are upper bounds for the L2-resident stages)."""
import csv, io, json, re, subprocess, sys

MAP = [  # (regex on the ncu kernel name, library profile label)
    (r"l2p(_tma|_warp)?_kernel", "l2p"), (r"vol_insert_kernel", "insert"), (r"insert_(sorted|heavy)_kernel", "insert"), (r"p2m_sorted_kernel", "p2m"),
    (r"brick_hist_kernel", "brick_hist"), (r"brick_(colscan|segsum|segscan|segfill|start|scan_small)_kernel", "brick_scan"),
    (r"brick_scatter(_rank)?_kernel", "brick_scatter"), (r"brick_p2m_kernel", "brick_p2m"),
    (r"cell_keys_kernel", "cell_keys"), (r"place_kernel", "sort_place"),
    (r"segment_sort_\w+_kernel", "sort_segments"), (r"scan_\w+_kernel", "scan"),
    (r"sep_pre_kernel", "m2l_sep_pre"), (r"sep_post_kernel", "m2l_sep_post_l2l"),
    (r"sep_pass_kernel<\d+, 0", "m2l_sep_z"), (r"sep_pass_kernel<\d+, 1", "m2l_sep_y"),
    (r"sep_pass_kernel<\d+, 2", "m2l_sep_x"), (r"m2l_tc_kernel", "m2l_tc_L4"),
    (r"m2l_ffma_kernel", "m2l_L3"), (r"m2l_reduce_kernel", "m2l_reduce"),
    (r"absmax_kernel", "m2l_absmax"), (r"split_\w+_kernel", "m2l_split"),
    (r"l2l_kernel", "l2l"), (r"m2m(_child)?_kernel", "m2m"), (r"weighted_grad_kernel", "wgrad_recycle"),
    (r"domain_check_kernel", "domain_check"),
]


def main():
    rep, steps, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = dict(zip(h, rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot, launches, dur = {}, {}, {}
    # the separable kernels also run the coarse levels' far tables on smaller
    # grids (labels m2l_sepfar_*): the finest level is the largest grid seen
    def cta_count(d):
        return eval(d.get("Grid Size", "(1,)").replace("(", "(").strip() or "(1,)")
    sep_max = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        if re.search(r"sep_(pre|post|pass)_kernel", d["Kernel Name"]):
            g = cta_count(d)
            n = g[0] * (g[1] if len(g) > 1 else 1) * (g[2] if len(g) > 2 else 1)
            fam = re.search(r"sep_(pre|post|pass)_kernel", d["Kernel Name"]).group(1)
            sep_max[fam] = max(sep_max.get(fam, 0), n)
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"]
        lab = next((l for pat, l in MAP if re.search(pat, name)), None)
        if lab is None:
            continue
        m = re.search(r"sep_(pre|post|pass)_kernel", name)
        if m:
            g = cta_count(d)
            n = g[0] * (g[1] if len(g) > 1 else 1) * (g[2] if len(g) > 2 else 1)
            if n < sep_max[m.group(1)]:
                lab = lab.replace("m2l_sep_", "m2l_sepfar_").replace("_post_l2l", "_post")
        b = sum(float(d[m].replace(",", "")) * scale[units[m]]
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        tot[lab] = tot.get(lab, 0.0) + b
        launches[lab] = launches.get(lab, 0) + 1
        t = float(d["gpu__time_duration.sum"].replace(",", ""))
        t *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(units["gpu__time_duration.sum"], 1e-3)
        dur[lab] = dur.get(lab, 0.0) + t
    res = {"source": f"ncu --set full --clock-control none, {rep.split('/')[-1]}, "
                     f"{steps:g} steps captured (cold-cache replays)",
           "bytes_per_step": {k: v / steps for k, v in tot.items()},
           "launches_per_step": {k: v / steps for k, v in launches.items()},
           "serial_ms_per_step": {k: v / steps for k, v in dur.items()}}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
