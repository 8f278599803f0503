"""DRAM bytes per launch of the render kernels from an .ncu-rep -> one JSON line (bench.py's roofline.traffic).
usage: traffic_json.py rep.ncu-rep kernel-name"""
import csv, io, json, re, subprocess, sys

rep, name = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    m = re.search(r"(render_fwd|render_bwd|cull)_kernel", d["Kernel Name"])
    if not m:
        continue
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(d[k].replace(",", "")) * scale[units[hdr.index(k)]]
    out[f"{m.group(1)}<{name}>"] = tot
print(json.dumps(out))
