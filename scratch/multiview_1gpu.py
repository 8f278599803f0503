"""BASELINE.json configs[3] as one rank sees it: 3 M primitives, 1920x1080, 64 orbit cameras sharded
over 8 ranks -> this rank's 8 views per iteration (view v -> rank v mod 8), gradients accumulated
over the views, one replicated Adam step.  One GPU, no collective (the all-reduce of the 14 N
float32 gradient buffer is reported as bytes).  Writes a markdown summary.
usage: multiview_1gpu.py out.md [--splats N] [--views-per-rank V]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_12369_b200 as d
from paper_2501_12369_b200 import synthetic as syn
from paper_2501_12369_b200.multiview import ViewParallelTrainer, bind_context, local_views

out = sys.argv[1]
n = int(sys.argv[sys.argv.index("--splats") + 1]) if "--splats" in sys.argv else 3_000_000
world, rank, n_views = 8, 0, 64
w, h = 1920, 1080
dev = torch.device("cuda", 0)
ctx = d.Context(0); st = torch.cuda.Stream(dev); torch.cuda.set_stream(st); ctx.use_torch_stream()
rows = []
for name in ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"]:
    k, psi = d.kernel_preset(name), d.default_psi(name)
    truth = syn.scene_b(n, 1); init = syn.perturb(truth, 2)
    truth_d = torch.from_numpy(truth).to(dev)
    views = local_views(n_views, world, rank)
    cams = {v: syn.orbit_camera(v, n_views, w, h, 1600.0) for v in views}
    targets = {}
    for v in views:
        t = torch.empty((h, w, 3), device=dev)
        ctx.evaluate_view(k, psi, truth_d, cams[v], (0, 0, 0), grad_image=torch.zeros_like(t), image_out=t)
        targets[v] = t
    params = torch.from_numpy(init).to(dev)
    lrs = torch.from_numpy(syn.learning_rates(init)).to(dev)
    ev, adam = bind_context(ctx, k, psi, cams, targets, want_loss=False)
    tr = ViewParallelTrainer(params, lrs, n_views, ev, adam, world=1, rank=0)
    tr.views = views  # this rank's share of the 64 cameras
    for _ in range(2):
        tr.step(want_loss=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 5
    a.record()
    for _ in range(iters):
        tr.step(want_loss=False)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    wc = ctx.work_counters()
    rows.append((name, ms, len(views) / (ms * 1e-3), wc["entries"]))
    del tr, params, targets, truth_d
    torch.cuda.empty_cache()
lines = ["# Round 1 - configs[3] as one rank sees it (one B200)", "",
         f"`scratch/multiview_1gpu.py`: {n:,} primitives, 1920x1080, 64 orbit cameras sharded view v -> rank v mod 8: this rank's 8 views "
         "per iteration through `ViewParallelTrainer` (gradients accumulated over the views, L1 + D-SSIM loss, one Adam step), device-resident, "
         "CUDA events, mean of 5 iterations after 2 warm-ups.  No collective runs here: the multi-rank iteration adds one all-reduce of the "
         f"14 N float32 gradient buffer ({14 * n * 4 / 1e6:.0f} MB) between the last view and the Adam step.", "",
         "| kernel | ms per iteration (8 views + Adam) | views/s on this rank | tile entries of the last view |", "|---|---|---|---|"]
for name, ms, vps, k_ in rows:
    lines.append(f"| {name} | {ms:.2f} | {vps:.1f} | {k_:,} |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
