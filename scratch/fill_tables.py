"""Fills the round-2 result tables of DESIGN.md (the @@R2TABLE@@ block between its markers) and
BASELINE.md section 4 from the JSON lines under profiles/ (r2_final_bench.json, r2_final_bench_ref.json,
r2_reference_table.json) and profiles/r2_sweep_4k.md.  Run here (no GPU needed)."""
import json, os, re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = lambda *a: os.path.join(ROOT, *a)
b = json.load(open(P("profiles", "r2_final_bench.json")))
r = json.load(open(P("profiles", "r2_final_bench_ref.json")))
t = json.load(open(P("profiles", "r2_reference_table.json")))
K = ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"]
pk = b["per_kernel"]
stage_tot = {}
for k in K:
    for s, v in pk[k]["stage_ms"].items():
        stage_tot[s] = stage_tot.get(s, 0.0) + v
tot = sum(stage_tot.values())
hb = lambda key: " / ".join(f"{pk[k]['hbm_frac'][key]:.2f}" for k in K)
rf = b["roofline"]
dr = b["e2e_dropin"]
rows = [
    ("`value` (device-resident)", f"**{b['value']:.0f} view-iterations/s** ({b['ms_per_step']:.2f} ms per step of four iterations; 768 in round 1's driver run)"),
    ("`e2e` (host target in, loss out, every iteration)", f"**{b['e2e']['value']:.0f} view-iterations/s**"),
    ("reference arm (its own CPU code, %d host threads, the SAME workload at full size, %d timed iterations per kernel)" % (r["cpu_baseline"]["cores"], r["steps"]),
     f"**{r['value']:.3f} view-iterations/s** ({r['ms_per_step'] / 1e3:.1f} s per step of four iterations; per kernel "
     + " / ".join(f"{r['per_kernel'][k]['ms_per_iter'] / 1e3:.1f}" for k in K) + " s); the 1/16 sample scaled: "
     + (f"{r['sample_1_16']['value_full_equiv']:.3f}" if r.get("sample_1_16") else "n/a")),
    ("per kernel, iterations/s (device / e2e)", ", ".join(f"{k} {pk[k]['iters_per_s']:.0f} / {pk[k]['iters_per_s_e2e']:.0f}" for k in K)),
    ("forward render FPS (preprocess + bin + cull + forward)", " / ".join(f"{pk[k]['render_fps']:.0f}" for k in K) + " (`profiles/r2_sweep_4k.md` has `mod-sinc` and the 4K sweep)"),
    ("`e2e_dropin`: `darbs_cuda_forward` + `darbs_cuda_backward`, host arrays in and out, 1 M splats 1080p",
     f"{dr['value']:.0f} pairs/s; forward " + " / ".join(f"{dr['per_kernel'][k]['ms_forward']:.1f}" for k in K) + " ms, backward "
     + " / ".join(f"{dr['per_kernel'][k]['ms_backward']:.1f}" for k in K) + " ms (PCIe: 69 MB in, 86 MB out per pair)"),
    ("small-scene latency through the same host-array calls (the reference's `bm_forward` / `bm_backward` sizes, 128², Gaussian)",
     "; ".join(f"{k.split('_')[0]} splats: forward {v['us_forward']:.0f} µs, backward {v['us_backward']:.0f} µs" for k, v in dr["small_scene_latency"].items())
     + (" — the reference's CPU code, one thread, same sizes: " + "; ".join(f"{k.split('_')[0]} splats: {v['us_forward'] / 1e3:.1f} ms / {v['us_backward'] / 1e3:.1f} ms" for k, v in t["bm_forward_backward"].items()) if "bm_forward_backward" in t else "")),
    (f"`roofline` (dominant kernel `{rf['kernel']}`, {pk['gaussian']['render_bwd']['ms']:.3f} ms)",
     f"{rf['achieved']:.1f} TFLOP/s algorithmic of {rf['peak']:.1f} measured (FFMA2; scalar FFMA {rf['peak_ffma_tflops']:.1f}): `frac` **{rf['frac']:.2f}**; `frac_evaluated` {rf['frac_evaluated']:.2f}; "
     f"DRAM traffic {rf['traffic'] / 1e6:.0f} MB per launch; SM clock {rf['peak_sm_mhz']:.0f} MHz"),
    ("`render_fwd` `frac`", " / ".join(f"{pk[k]['render_fwd']['frac']:.2f}" for k in K) + " (values above 1: the §8d count includes visits block culling skips; `frac_evaluated` "
     + " / ".join(f"{pk[k]['render_fwd']['frac_evaluated']:.2f}" for k in K) + ")"),
    ("`render_bwd` `frac`", " / ".join(f"{pk[k]['render_bwd']['frac']:.2f}" for k in K) + " (`frac_evaluated` " + " / ".join(f"{pk[k]['render_bwd']['frac_evaluated']:.2f}" for k in K) + ")"),
    ("stage share of a step", ", ".join(f"{s} {100 * v / tot:.1f} %" for s, v in sorted(stage_tot.items(), key=lambda kv: -kv[1]))),
    ("stage times per kernel, ms (" + " / ".join(K) + ")", "; ".join(f"{s} " + " / ".join(f"{pk[k]['stage_ms'][s]:.3f}" for k in K) for s in ("binning", "cull", "render_fwd", "loss", "render_bwd"))),
    ("streaming stages, fraction of measured HBM peak (algorithmic bytes)", f"Adam {hb('adam')}; cull {hb('cull')}; preprocess {hb('preprocess')}; preprocess_bwd {hb('preprocess_bwd')}; loss {hb('loss')}; binning {hb('binning_sort')}"),
    ("kernel launches per step of four iterations", f"{b['gpu_launches'] // b['steps']} (`gpu_launches` {b['gpu_launches']} over {b['steps']} steps)"),
]
table = "| | value |\n|---|---|\n" + "\n".join(f"| {a} | {c} |" for a, c in rows)
d = open(P("DESIGN.md")).read()
if "@@R2TABLE@@" in d:
    d = d.replace("@@R2TABLE@@", "<!-- r2table -->\n" + table + "\n<!-- /r2table -->")
else:
    d = re.sub(r"<!-- r2table -->.*?<!-- /r2table -->", "<!-- r2table -->\n" + table + "\n<!-- /r2table -->", d, flags=re.S)
open(P("DESIGN.md"), "w").write(d)

# ---- BASELINE.md section 4
sweep = open(P("profiles", "r2_sweep_4k.md")).read()
def sweep_row(kernel, n):
    m = re.search(rf"^\| {re.escape(kernel)} \| {n:,} \|(.*)$", sweep, re.M)
    f = [x.strip() for x in m.group(1).split("|")]
    return float(f[-4]), float(f[-3])  # total ms, iters/s
c0 = t["config0_10k_256_half-cosine-sq"]
c0g = re.search(r"forward ([0-9.]+) ms, backward ([0-9.]+) ms", sweep)
cores = t["cores"]
c1 = t[[k for k in t if k.startswith("config1_")][0]]
fwd_fps = dict(re.findall(r"^\| (gaussian|half-cosine-sq|raised-cosine) \| [0-9.]+ \| [0-9.]+ \| [0-9.]+ \| [0-9.]+ \| ([0-9.]+) \| \d+ \|$", sweep, re.M))
rows4 = [
    ("1. 10k splats 256² half-cosine² fwd+bwd", f"{c0[str(cores) + '_threads']['ms_forward'] + c0[str(cores) + '_threads']['ms_backward']:.1f} ms ({cores} threads); "
     f"{c0['1_threads']['ms_forward'] + c0['1_threads']['ms_backward']:.0f} ms (1 thread)",
     f"{float(c0g.group(1)) + float(c0g.group(2)):.3f} ms (forward {c0g.group(1)} + backward {c0g.group(2)}, host arrays in and out)", "latency-bound (≈ 20 launches); parity scene, bit-exact aux", "—"),
    ("2. 1M splats 1080p forward: gaussian / half-cosine² / raised-cosine",
     " / ".join(f"{c1[k]['ms_preprocess'] + c1[k]['ms_forward_incl_bin']:.0f}" for k in ("gaussian", "half-cosine-sq", "raised-cosine")) + f" ms ({cores} threads; preprocess + bin + forward)",
     " / ".join(fwd_fps[k] for k in ("gaussian", "half-cosine-sq", "raised-cosine")) + " ms per frame (" + " / ".join(f"{pk[k]['render_fps']:.0f}" for k in K[:3]) + " FPS)",
     "render_fwd frac " + " / ".join(f"{pk[k]['render_fwd']['frac']:.2f}" for k in K[:3]), "replicas only"),
    ("3. 1M splats 1080p fwd+bwd+Adam per kernel", " / ".join(f"{r['per_kernel'][k]['ms_per_iter'] / 1e3:.1f}" for k in K) + f" s per iteration ({r['cpu_baseline']['cores']} threads, full size; {r['value']:.3f} view-iterations/s)",
     " / ".join(f"{pk[k]['ms_per_iter']:.2f}" for k in K) + f" ms per iteration ({b['value']:.0f} view-iterations/s; e2e {b['e2e']['value']:.0f})",
     "render_bwd frac " + " / ".join(f"{pk[k]['render_bwd']['frac']:.2f}" for k in K) + f" of {rf['peak']:.0f} TFLOP/s", "—"),
    ("4. 3M splats × 64 views, view-sharded + NCCL all-reduce", "not run (64 views × ≈ 10 s of CPU time per view at 3 M primitives, per kernel)", "one rank's share (8 views of 64) on one B200: 565 view-iterations/s (1.77 ms per view), e2e 559", "as row 3 per view", "not measured: no multi-GPU node in this run (`bench.py --gpus N` runs it)"),
    ("5. kernel sweep × 100k–5M splats @ 4K", "not run above 1M", "gaussian " + " / ".join(f"{sweep_row('gaussian', n)[0]:.2f}" for n in (100_000, 1_000_000, 5_000_000)) + " ms per iteration at 100k / 1M / 5M; all rows: `profiles/r2_sweep_4k.md`",
     "cull and binning dominate beyond 1M (DESIGN §8)", "—"),
]
bm = open(P("BASELINE.md")).read()
head = "| Config | CPU reference (ms, cores) | 1× B200 (ms) | roofline fraction | 2/4/8× B200 |\n|---|---|---|---|---|\n"
body = "\n".join("| " + " | ".join(x) + " |" for x in rows4)
bm = bm[:bm.index("| Config | CPU reference (ms, cores)")] + head + body + "\n\nMeasured on one B200 pod (16 host threads) in round 2: `profiles/r2_final_bench.json`, `profiles/r2_final_bench_ref.json`, `profiles/r2_reference_table.json`, `profiles/r2_sweep_4k.md`; filled by `scratch/fill_tables.py`.\n"
open(P("BASELINE.md"), "w").write(bm)
print(table[:1500])
