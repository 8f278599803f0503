"""Turns an `ncu --metrics gpu__time_duration.sum --csv` log into the launch-list markdown under
profiles/.  usage: launch_list.py in.csv out.md "title" [first-kernel-substring]"""
import csv, sys
from collections import OrderedDict

src, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
first = sys.argv[4] if len(sys.argv) > 4 else None
rows = list(csv.reader(open(src, errors="replace")))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
launches = []
for r in rows[h + 1:]:
    if len(r) != len(hdr):
        continue
    v = float(r[iv].replace(",", ""))
    v = v / 1e3 if r[iu] in ("ns", "nsecond") else v * 1e3 if r[iu] in ("ms", "msecond") else v
    launches.append((r[ik], v))
if first:
    starts = [i for i, (k, _) in enumerate(launches) if first in k]
    if len(starts) >= 2:
        launches = launches[starts[0]:starts[1]]   # exactly one iteration
    elif starts:
        launches = launches[starts[0]:]
    last = [i for i, (k, _) in enumerate(launches) if "adam_kernel" in k]
    if last:
        launches = launches[:last[0] + 1]           # ... up to and including its Adam step
short = lambda k: k.replace("darbs_b200::<unnamed>::", "").replace("void ", "")[:72]
tot = sum(v for _, v in launches)
lines = [f"# {title}", "", f"{len(launches)} launches, {tot:.1f} us under ncu (per-launch times are cold-cache and serialised: "
         "compare SHARES with the stage times `bench.py` measures with CUDA events, not absolutes).", "",
         "| # | kernel | us | share |", "|---|---|---|---|"]
for i, (k, v) in enumerate(launches):
    lines.append(f"| {i} | `{short(k)}` | {v:.1f} | {100 * v / tot:.1f}% |")
agg = OrderedDict()
for k, v in launches:
    agg[short(k)] = agg.get(short(k), 0.0) + v
lines += ["", "| kernel (summed) | us | share |", "|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda t: -t[1]):
    lines.append(f"| `{k}` | {v:.1f} | {100 * v / tot:.1f}% |")
open(out, "w").write("\n".join(lines) + "\n")
print("wrote", out, len(launches), "launches", f"{tot:.1f} us")
