"""Turns an .ncu-rep (read here, no GPU) into the markdown summary committed under profiles/.
usage: make_profile_summary.py rep.ncu-rep out.md "title" [kernel-regex]"""
import csv, io, re, subprocess, sys

rep, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
kre = sys.argv[4] if len(sys.argv) > 4 else "."
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"), ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (registers), CTAs/SM"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (shared), CTAs/SM"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / instruction"),
    ("sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "L1 wavefronts, shared"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"), ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("lts__t_sectors_op_red.sum", "L2 sectors, reductions (red.global)"),
    ("lts__t_sectors_op_atom.sum", "L2 sectors, atomics with return (atom.global)"),
    ("smsp__inst_executed_op_global_red.sum", "warp instructions, red.global"),
    ("smsp__inst_executed_op_global_atom.sum", "warp instructions, atom.global"),
    ("smsp__inst_executed_op_shared_atom.sum", "warp instructions, shared-memory atomics"),
    ("l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum", "L1 set accesses, red.global"),
]


def derived(d, units, hdr):
    """achieved DRAM GB/s and reduction / atomic throughput: counter / kernel duration"""
    def num(k):
        try:
            return float(d[k].replace(",", ""))
        except (KeyError, ValueError):
            return None

    def in_unit(k, scale):
        v = num(k)
        if v is None:
            return None
        u = units[hdr.index(k)]
        return v * scale.get(u, 1.0)

    dur = in_unit("gpu__time_duration.sum", {"us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1.0, "second": 1.0})
    if not dur:
        return []
    byt = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd, wr = in_unit("dram__bytes_read.sum", byt), in_unit("dram__bytes_write.sum", byt)
    out = []
    if rd is not None and wr is not None:
        out.append(f"| **achieved HBM traffic** | {(rd + wr) / dur / 1e9:,.0f} GB/s ({(rd + wr) / 1e6:,.1f} MB in {dur * 1e6:,.1f} us) |")
    red, atom = num("lts__t_sectors_op_red.sum"), num("lts__t_sectors_op_atom.sum")
    if red is not None and (red or atom):
        out.append(f"| **atomic throughput at L2** | {red / dur / 1e9:,.2f} G red-sectors/s"
                   + (f", {atom / dur / 1e9:,.2f} G atom-sectors/s" if atom else "") + " |")
    ri = num("smsp__inst_executed_op_global_red.sum")
    if ri:
        out.append(f"| red.global warp instructions per second | {ri / dur / 1e9:,.3f} G/s |")
    return out

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
lines = [f"# {title}", "", f"Source: `{rep}` (ncu --set full --clock-control none --import-source on, one B200; "
         "times under ncu are cold-cache and serialised — use them for shares and counters, not as bench values).", ""]
seen = set()
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"]
    if not re.search(kre, name) or name in seen:
        continue
    seen.add(name)
    lines += [f"## `{name[:140]}`", "", "| metric | value |", "|---|---|"]
    for k, label in KEYS:
        if k in d and d[k] != "":
            v = d[k]
            try:
                v = f"{float(v.replace(',', '')):,.2f}".rstrip("0").rstrip(".")
            except ValueError:
                pass
            lines.append(f"| {label} | {v} {units[hdr.index(k)]} |")
    lines += derived(d, units, hdr)
    lines.append("")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
done = set()
for b in re.split(r'(?m)^"Kernel Name",', src)[1:]:
    ls = list(csv.reader(io.StringIO(b)))
    name = ls[0][0]
    if name in done or not re.search(kre, name):
        continue
    done.add(name)
    h = ls[1]
    data = [r for r in ls[2:] if len(r) == len(h) and r[0].startswith("0x")]
    if not data:
        continue
    ts = sum(int(r[h.index("# Samples")]) for r in data) or 1
    stalls = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    agg = sorted(((sum(int(r[h.index(x)]) for r in data), x[6:]) for x in stalls), reverse=True)[:8]
    lines += [f"### warp-state samples, `{name[:100]}`", "",
              ", ".join(f"{n} {100 * v / ts:.1f}%" for v, n in agg), ""]
    # top instructions by samples
    ia, isamp, isrc = h.index("Instructions Executed"), h.index("# Samples"), h.index("Source")
    top = sorted(data, key=lambda r: -int(r[isamp]))[:12]
    lines += ["| samples % | executed | SASS |", "|---|---|---|"]
    for r in top:
        lines.append(f"| {100 * int(r[isamp]) / ts:.2f} | {int(r[ia]):,} | `{r[isrc].strip()[:80]}` |")
    lines.append("")
open(out, "w").write("\n".join(lines))
print("wrote", out, len(lines), "lines")
