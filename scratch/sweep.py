"""BASELINE.json configs[4] and configs[1]: DARBF kernel sweep (gaussian, half-cosine-sq,
raised-cosine, inv-multiquadratic) x splat count at 3840x2160 (full training iteration, scene B
scaled to 4K with focal 3200), and forward-only render FPS at 1M splats 1080p.  Device-resident,
CUDA-event stage times (median of 5 after 2 warm-ups).  Writes a markdown table.
usage: sweep.py out.md [--quick]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_12369_b200 as d
from paper_2501_12369_b200 import synthetic as syn

out = sys.argv[1]
quick = "--quick" in sys.argv
KERNELS = ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"]
dev = torch.device("cuda", 0)
ctx = d.Context(0); st = torch.cuda.Stream(dev); torch.cuda.set_stream(st); ctx.use_torch_stream()
ctx.set_stage_timing(True)
STAGES = ["preprocess", "binning", "cull", "render_fwd", "loss", "render_bwd", "preprocess_bwd", "adam"]


def run(name, n, w, h, focal, reps=5):
    k, psi = d.kernel_preset(name), d.default_psi(name)
    truth = syn.scene_b(n, 1); init = syn.perturb(truth, 2)
    cam = syn.orbit_camera(0, 1, w, h, focal)
    lrs = torch.from_numpy(syn.learning_rates(init).reshape(-1)).to(dev)
    target = torch.empty((h, w, 3), device=dev)
    ctx.evaluate_view(k, psi, torch.from_numpy(truth).to(dev), cam, (0, 0, 0), grad_image=torch.zeros_like(target), image_out=target)
    p = torch.from_numpy(init).to(dev); g = torch.zeros_like(p)
    m = torch.zeros(14 * n, device=dev); v = torch.zeros(14 * n, device=dev)
    rows = []
    for it in range(reps + 2):
        g.zero_()
        ctx.evaluate_view(k, psi, p, cam, (0, 0, 0), target=target, lam=0.2, param_grads=g)
        t = ctx.stage_times()
        ctx.adam_step(p.view(-1), g.view(-1), m, v, lrs, it + 1)
        t["adam"] = ctx.stage_times()["adam"]
        if it >= 2:
            rows.append([t[s] for s in STAGES])
    med = np.median(np.array(rows), axis=0)
    wc = ctx.work_counters()
    del p, g, m, v, target, lrs
    torch.cuda.empty_cache()
    return dict(zip(STAGES, med)), wc


lines = ["# Round 2 - DARBF kernel sweep at 3840x2160, forward render FPS at 1080p, and the 10 k-splat case (one B200)", "",
         "`scratch/sweep.py`: device-resident, CUDA-event stage times, median of 5 after 2 warm-ups; BASELINE.json `configs[4]`, `configs[1]`, `configs[0]`.", "",
         "Scene B of bench.py scaled to the resolution (focal 3200 at 4K), one orbit view, full training iteration "
         "(preprocess, bin+sort, cull, render fwd, L1 + D-SSIM loss, render bwd, preprocess bwd, Adam); "
         "stage times in ms, median of 5.", "",
         "| kernel | splats | tile entries K | visits V | " + " | ".join(STAGES) + " | total ms | iters/s | fwd-only FPS |",
         "|---|---|---|---|" + "---|" * (len(STAGES) + 3)]
counts = [100_000, 1_000_000] if quick else [100_000, 300_000, 1_000_000, 3_000_000, 5_000_000]
for name in KERNELS:
    for n in counts:
        t, wc = run(name, n, 3840, 2160, 3200.0)
        tot = sum(t.values())
        fps = 1e3 / (t["preprocess"] + t["binning"] + t["cull"] + t["render_fwd"])
        lines.append(f"| {name} | {n:,} | {wc['entries']:,} | {wc['visits']:,} | " + " | ".join(f"{t[s]:.3f}" for s in STAGES)
                     + f" | {tot:.3f} | {1e3 / tot:.1f} | {fps:.0f} |")
        print(lines[-1], flush=True)
lines += ["", "## Forward render, 1,000,000 splats, 1920x1080 (BASELINE.json configs[1])", "",
          "| kernel | preprocess | binning | cull | render_fwd | frame ms | FPS |", "|---|---|---|---|---|---|---|"]
for name in KERNELS + ["mod-sinc"]:
    t, wc = run(name, 1_000_000, 1920, 1080, 1600.0)
    ms = t["preprocess"] + t["binning"] + t["cull"] + t["render_fwd"]
    lines.append(f"| {name} | {t['preprocess']:.3f} | {t['binning']:.3f} | {t['cull']:.3f} | {t['render_fwd']:.3f} | {ms:.3f} | {1e3 / ms:.0f} |")
    print(lines[-1], flush=True)
# configs[0]: 10 k random splats (input A), 256 x 256, half-cosine-sq, forward + backward through the host-pointer ABI
import time
sc = syn.scene_a(10_000, 256, 256, 0)
k = d.kernel_preset("half-cosine-sq")
arrs = [sc[key] for key in ("mu2", "conic", "radius", "depth", "opacity", "rgb")]
g = np.ones((256, 256, 3), np.float32)
ctx.set_stage_timing(False)
tf = tb = 0.0
for rep in range(55):
    t0 = time.perf_counter(); ctx.forward(k, *arrs, 256, 256, (0.1, 0.2, 0.3)); t1 = time.perf_counter()
    ctx.backward(k, g, 10_000); t2 = time.perf_counter()
    if rep >= 5:
        tf += (t1 - t0) / 50; tb += (t2 - t1) / 50
lines += ["", "## 10,000 random splats, 256x256, half-cosine-sq, forward + backward (BASELINE.json configs[0])", "",
          f"Host arrays in and out through darbs_cuda_forward / darbs_cuda_backward (all copies inside the calls), mean of 50: "
          f"forward {1e3 * tf:.3f} ms, backward {1e3 * tb:.3f} ms."]
open(out, "w").write("\n".join(lines) + "\n")
