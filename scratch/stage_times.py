"""Per-stage device times of one training iteration per kernel (CUDA-event stage timers of the library)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2501_12369_b200 as darbs  # noqa: E402
from paper_2501_12369_b200 import synthetic as syn  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
w, h = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1920, 1080)
names = sys.argv[4:] or ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"]
dev = torch.device("cuda", 0)
ctx = darbs.Context(0)
ctx.use_torch_stream()
truth = syn.scene_b(n, 1)
init = syn.perturb(truth, 2)
cam = syn.orbit_camera(0, 1, w, h, 1600.0 * w / 1920)
truth_d = torch.from_numpy(truth).to(dev)
lrs = torch.from_numpy(syn.learning_rates(init).reshape(-1)).to(dev)
for name in names:
    k, psi = darbs.kernel_preset(name), darbs.default_psi(name)
    target = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    ctx.evaluate_view(k, psi, truth_d, cam, (0, 0, 0), grad_image=torch.zeros_like(target), image_out=target)
    params = torch.from_numpy(init).to(dev)
    grads = torch.zeros((n, 14), device=dev)
    m, v = torch.zeros(14 * n, device=dev), torch.zeros(14 * n, device=dev)
    for _ in range(3):
        ctx.evaluate_view(k, psi, params, cam, (0, 0, 0), target=target, lam=0.2, param_grads=grads, accumulate=False)
    ctx.set_stage_timing(True)
    acc = None
    reps = 5
    for _ in range(reps):
        ctx.evaluate_view(k, psi, params, cam, (0, 0, 0), target=target, lam=0.2, param_grads=grads, accumulate=False)
        st = ctx.stage_times()
        ctx.adam_step(params.view(-1), grads.view(-1), m, v, lrs, 1)
        st["adam"] = ctx.stage_times()["adam"]
        acc = st if acc is None else {kk: acc[kk] + st[kk] for kk in st}
    ctx.set_stage_timing(False)
    wc = ctx.work_counters()
    print(name, {kk: round(1e3 * vv / reps, 1) for kk, vv in acc.items()}, "us; total",
          round(1e3 * sum(acc.values()) / reps, 1), "entries", wc["entries"], "survivors", wc["survivors"], flush=True)
