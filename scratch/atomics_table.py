"""gpurun_out/r2_atomics_<kernel>.csv (scratch/prof_atomics.sh) -> profiles/r2_atomics.md"""
import csv, glob, os, re

def num(s):
    try:
        return float(s.replace(',', ''))
    except ValueError:
        return 0.0

rows_out = []
for f in sorted(glob.glob('gpurun_out/r2_atomics_*.csv')):
    name = os.path.basename(f)[len('r2_atomics_'):-4]
    rows = list(csv.reader(open(f, errors='replace')))
    h = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
    hdr = rows[h]
    ik, im, iu, iv = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Unit'), hdr.index('Metric Value')
    per = {}
    for r in rows[h + 1:]:
        if len(r) == len(hdr):
            per.setdefault((r[0], r[ik]), {})[r[im]] = (num(r[iv]), r[iu])
    seen = set()
    for (_id, k), m in per.items():
        short = re.sub(r'\(.*', '', k.replace('darbs_b200::', '').replace('<unnamed>::', '').replace('void ', ''))
        if short in seen:
            continue
        seen.add(short)
        dur = m['gpu__time_duration.sum']
        d = dur[0] * {'us': 1e-6, 'usecond': 1e-6, 'ns': 1e-9, 'nsecond': 1e-9, 'ms': 1e-3, 'msecond': 1e-3}.get(dur[1], 1e-6)
        g = lambda n: m.get(n, (0.0, ''))[0]
        byt = lambda n: g(n) * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(m.get(n, (0, 'byte'))[1], 1)
        red, atom = g('lts__t_sectors_op_red.sum'), g('lts__t_sectors_op_atom.sum')
        rows_out.append((name, short, d * 1e6, g('smsp__inst_executed_op_global_red.sum'), g('smsp__inst_executed_op_global_atom.sum'),
                         red, atom, (red + atom) / d / 1e9, (byt('dram__bytes_read.sum') + byt('dram__bytes_write.sum')) / d / 1e9,
                         g('smsp__inst_executed_op_shared_atom.sum')))
out = ["# Round 2 - atomic / reduction throughput and achieved HBM GB/s per kernel", "",
       "`scratch/prof_atomics.sh` on one B200: `ncu --metrics lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,"
       "smsp__inst_executed_op_global_red.sum,... --clock-control none` over one training iteration per DARBF kernel "
       "(scene B, 1 M primitives, 1080p). L2 sectors are 32 B; a lane's `red.global.add.v4.f32` is one sector. Times "
       "under ncu are serialised and cold-cache.", "",
       "| DARBF kernel | kernel | us | red.global warp instr. | atom.global warp instr. | L2 red sectors | L2 atom sectors | "
       "G atomic sectors/s | achieved HBM GB/s | shared-memory atomic warp instr. |", "|---|---|---|---|---|---|---|---|---|---|"]
for r in rows_out:
    out.append(f"| {r[0]} | `{r[1]}` | {r[2]:.1f} | {r[3]:,.0f} | {r[4]:,.0f} | {r[5]:,.0f} | {r[6]:,.0f} | {r[7]:.2f} | {r[8]:,.0f} | {r[9]:,.0f} |")
open('profiles/r2_atomics.md', 'w').write("\n".join(out) + "\n")
print("\n".join(out[4:20]))
