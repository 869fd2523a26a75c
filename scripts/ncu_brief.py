"""Brief per-kernel table from an ncu report: python scripts/ncu_brief.py REP [regex]"""
import csv, io, re, subprocess, sys
M = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,"
     "sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,"
     "sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,"
     "smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,launch__registers_per_thread,"
     "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,"
     "smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,"
     "smsp__average_warp_latency_issue_stalled_lg_throttle.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", M],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"]
    if pat and not pat.search(name):
        continue
    short = re.sub(r"\(.*", "", name).replace("void ", "").replace("unnamed>::", "")[:40]
    vals = []
    for m in M.split(","):
        v = d.get(m, "")
        key = m.split("__", 1)[1].replace(".avg.pct_of_peak_sustained_", "%").replace("average_warp_latency_issue_stalled_", "st_")[:28]
        vals.append(f"{key}={v}")
    print(short, " ".join(vals))
