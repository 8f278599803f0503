"""Summarise an .ncu-rep (read here, no GPU): key raw metrics per kernel and a per-region
instruction / stall breakdown from the source page.  usage: ncu_summary.py rep [kernel-regex]"""
import csv, subprocess, sys, io, re

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
WANT = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
        "lts__t_bytes.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__cycles_active.avg", "sm__cycles_elapsed.max"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if not re.search(kre, d["Kernel Name"]):
        continue
    print("=====", d["Kernel Name"][:110])
    for k in WANT:
        if k in d:
            print(f"  {k:70s} {d[k]:>18s} {units[hdr.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre],
                     capture_output=True, text=True).stdout
# split per kernel
blocks = re.split(r'(?m)^"Kernel Name",', src)
for b in blocks[1:]:
    lines = list(csv.reader(io.StringIO(b)))
    name = lines[0][0]
    h = lines[1]
    data = [r for r in lines[2:] if len(r) == len(h) and r[0].startswith("0x")]
    ia, isamp, isrc, iaddr = h.index("Instructions Executed"), h.index("# Samples"), h.index("Source"), h.index("Address")
    tot = sum(int(r[ia]) for r in data)
    ts = sum(int(r[isamp]) for r in data) or 1
    print("=====", name[:110], f"inst {tot/1e6:.1f}M samples {ts}")
    stalls = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    agg = {x: sum(int(r[h.index(x)]) for r in data) for x in stalls}
    print("  stalls:", ", ".join(f"{k[6:]} {100*v/ts:.1f}%" for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
    if "--list" in sys.argv:
        base = int(data[0][iaddr], 16)
        for r in data:
            c = int(r[ia])
            if c > tot / 2000:
                print(f"   {int(r[iaddr],16)-base:6x} {c/1e6:8.2f}M {100*int(r[isamp])/ts:5.2f}%  {r[isrc].strip()[:90]}")
