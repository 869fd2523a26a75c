"""Instruction-count / stall hot spots of one kernel from an ncu source-page
export (`ncu -i R --page source --csv --print-source sass --kernel-name K`):
consecutive SASS lines with equal execution counts form a basic block.
    python scripts/ncu_sass_groups.py SASS.csv [min_share]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
h = rows[1]
ia, isrc, iex, ist = (h.index(k) for k in ("Address", "Source", "Instructions Executed",
                                            "Warp Stall Sampling (All Samples)"))
data = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    try:
        ex = float(r[iex].replace(",", ""))
    except ValueError:
        continue
    data.append((ex, float(r[ist].replace(",", "") or 0), r[ia], r[isrc]))
if len(data) > 10 and data[0][2] == data[len(data) // 2][2]:
    data = data[:len(data) // 2]
groups = []
for ex, st, a, src in data:
    if groups and groups[-1][0] == ex:
        g = groups[-1]
        g[1] += 1
        g[2] += st
        g[4].append(src.strip())
    else:
        groups.append([ex, 1, st, a, [src.strip()]])
tot = sum(g[0] * g[1] for g in groups)
stt = sum(g[2] for g in groups) or 1
print(f"total warp instructions {tot:.0f}, stall samples {stt:.0f}")
for g in groups:
    if g[0] * g[1] > thr * tot or g[2] > 2 * thr * stt:
        ops = " | ".join(x.split()[0] if not x.startswith("@") else x.split()[1] for x in g[4][:14])
        print(f"{g[0]:10.0f} x{g[1]:4d} = {g[0] * g[1] / tot * 100:5.1f}% instr, "
              f"{g[2] / stt * 100:5.1f}% stalls  {g[3]}  {ops}")
