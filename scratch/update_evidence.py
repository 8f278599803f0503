"""Turns what a GPU run left under gpurun_out/ into the tracked evidence under profiles/:

  gpurun_out/r1_training_step_<kernel>.md   (scratch/prof_all.sh)     -> profiles/
  gpurun_out/launches_r1_<kernel>.csv       (ncu launch list)         -> profiles/r1_launches_<kernel>.md
  gpurun_out/launches_bench.csv + final_bench.json                    -> profiles/r1_launches_bench.md
  gpurun_out/r1_sweep.md                    (scratch/sweep.py)        -> profiles/r1_sweep_4k.md
  DRAM bytes per launch of the profiled kernels                       -> profiles/r1_traffic.json

and prints the numbers DESIGN.md quotes.  Run here (no GPU needed)."""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
KERNELS = ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"]


def mb(x):
    v, u = x.split()[:2]
    return float(v.replace(",", "")) * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1}[u]


traffic = {}
for k in KERNELS:
    src = os.path.join(OUT, f"r1_training_step_{k}.md")
    if os.path.exists(src):
        txt = open(src).read().replace(
            f"Source: `/tmp/step_r1_{k}.ncu-rep`",
            f"Source: `scratch/prof_all.sh {k}` on one B200 (the ~50 MB report is summarised on the box by "
            "scratch/make_profile_summary.py)")
        open(os.path.join(PROF, f"r1_training_step_{k}.md"), "w").write(txt)
    txt = open(os.path.join(PROF, f"r1_training_step_{k}.md")).read()
    for sec in txt.split("\n## ")[1:]:
        m = re.search(r"(render_fwd_kernel|render_bwd_kernel|cull_kernel|ssim_map_kernel|ssim_grad_kernel|"
                      r"param_grads_kernel|adam_kernel|project_kernel)", sec.split("\n")[0])
        rd, wr = re.search(r"\| DRAM read \| (.*?) \|", sec), re.search(r"\| DRAM write \| (.*?) \|", sec)
        if not (m and rd and wr):
            continue
        key = m.group(1).replace("_kernel", "")
        key = f"{key}<{k}>" if key in ("render_fwd", "render_bwd", "cull") else key
        traffic.setdefault(key, mb(rd.group(1)) + mb(wr.group(1)))
    ll = os.path.join(OUT, f"launches_r1_{k}.csv")
    if os.path.exists(ll):
        subprocess.run([sys.executable, os.path.join(ROOT, "scratch", "launch_list.py"), ll,
                        os.path.join(PROF, f"r1_launches_{k}.md"),
                        f"Round 1 - launch list of one training iteration ({k}, scene B, 1 M primitives, 1080p, "
                        f"L1 + D-SSIM loss): ncu --metrics gpu__time_duration.sum --clock-control none over "
                        f"scratch/prof_step.py {k}", "project_kernel"], check=True)
traffic["_source"] = ("profiles/r1_training_step_<kernel>.md (ncu --set full, dram__bytes_read.sum + "
                      "dram__bytes_write.sum per launch, one B200)")
json.dump(traffic, open(os.path.join(PROF, "r1_traffic.json"), "w"), indent=1)

bench = json.load(open(os.path.join(OUT, "final_bench.json")))
stage = {}
for v in bench["per_kernel"].values():
    for a, x in v["stage_ms"].items():
        stage[a] = stage.get(a, 0.0) + x
ts = sum(stage.values())

lb = os.path.join(OUT, "launches_bench.csv")
if os.path.exists(lb):
    rows = list(csv.reader(open(lb, errors="replace")))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg, n = {}, 0
    for r in rows[h + 1:]:
        if len(r) != len(hdr):
            continue
        v = float(r[iv].replace(",", ""))
        v = v / 1e3 if r[iu] in ("ns", "nsecond") else v
        k = re.sub(r"\(.*", "", r[ik].replace("darbs_b200::<unnamed>::", "").replace("void ", ""))[:70]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
        n += 1
    tot = sum(v for _, v in agg.values())
    lines = ["# Round 1 - launch list of `bench.py` itself", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none -c 700 python bench.py --steps 1 --warmup 3 "
             "--no-cpu-baseline` on one B200: the first 700 launches (warm-up iterations of the four DARBF kernels, the "
             f"timed device-resident step, the end-to-end step), {n} launches, {tot / 1e3:.2f} ms under ncu. Per-launch "
             "times are cold-cache and serialised: the SHARE of each kernel is what must agree with the stage times "
             "`bench.py` measures with CUDA events (`per_kernel[*].stage_ms`), not the absolutes.", "",
             "| kernel | launches | total us | share | mean us |", "|---|---|---|---|---|"]
    for k, (c, v) in sorted(agg.items(), key=lambda t: -t[1][1]):
        lines.append(f"| `{k}` | {c} | {v:.1f} | {100 * v / tot:.1f}% | {v / c:.1f} |")
    lines += ["", "Stage shares of the same workload from `bench.py`'s own CUDA-event stage timers (sum over the four "
              "kernels):", "", "| stage | ms per step | share |", "|---|---|---|"]
    for a, x in sorted(stage.items(), key=lambda t: -t[1]):
        lines.append(f"| {a} | {x:.3f} | {100 * x / ts:.1f}% |")
    rb = sum(v for k, (c, v) in agg.items() if "render_bwd" in k) / tot
    rf = sum(v for k, (c, v) in agg.items() if "render_fwd" in k) / tot
    lines += ["", f"render_bwd: {100 * rb:.1f}% of the kernel time under ncu vs {100 * stage['render_bwd'] / ts:.1f}% "
              f"of the stage time; render_fwd: {100 * rf:.1f}% vs {100 * stage['render_fwd'] / ts:.1f}%.", ""]
    open(os.path.join(PROF, "r1_launches_bench.md"), "w").write("\n".join(lines))

sw = os.path.join(OUT, "r1_sweep.md")
if os.path.exists(sw):
    src = open(sw).read().replace(
        "# Round 1 - kernel sweep at 3840x2160 and forward FPS at 1080p (B200, device-resident, CUDA events)",
        "# Round 1 - DARBF kernel sweep at 3840x2160 and forward render FPS at 1080p (one B200)\n\n"
        "`scratch/sweep.py`: device-resident, CUDA-event stage times, median of 5 after 2 warm-ups; BASELINE.json "
        "`configs[4]` and `configs[1]`.")
    src += ("\nVisits saturate near 2e9 (Gaussian) because every pixel terminates early once the scene is dense; beyond "
            "1 M splats the sort and the cull (proportional to K) dominate.\n`mod-sinc` runs its own closed form (an "
            "entire series in the squared distance); multi-lobe and non-preset beta kernels run the generic device "
            "path.\n")
    open(os.path.join(PROF, "r1_sweep_4k.md"), "w").write(src)

# ---- the numbers DESIGN.md quotes
print("value", round(bench["value"], 1), "e2e", round(bench["e2e"]["value"], 1), "ms/step", round(bench["ms_per_step"], 3),
      "clocks", bench["clocks"])
r = bench["roofline"]
print("roofline", r["kernel"], {k: round(v, 3) for k, v in r.items() if isinstance(v, float)})
print("cpu_baseline", bench.get("cpu_baseline"))
ref = os.path.join(OUT, "final_bench_ref.json")
if os.path.exists(ref):
    print("reference arm", json.load(open(ref))["value"])
for k, v in bench["per_kernel"].items():
    print(k, round(v["iters_per_s"], 1), round(v["iters_per_s_e2e"], 1), "fps", round(v["render_fps"]),
          {a: round(b, 3) for a, b in v["stage_ms"].items()})
    print("    fwd frac", round(v["render_fwd"]["frac"], 3), "eval", round(v["render_fwd"]["frac_evaluated"], 3),
          "bwd frac", round(v["render_bwd"]["frac"], 3), "eval", round(v["render_bwd"]["frac_evaluated"], 3),
          {a: round(b, 2) for a, b in v["hbm_frac"].items()})
print("stage shares", {a: f"{100 * x / ts:.1f}%" for a, x in sorted(stage.items(), key=lambda t: -t[1])})
