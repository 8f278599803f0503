"""A few full training iterations (evaluate_view + adam) of one DARBF kernel on scene B, 1M primitives
1080p: the command ncu wraps for the per-kernel captures of the streaming stages."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2501_12369_b200 as d
from paper_2501_12369_b200 import synthetic as syn
name = sys.argv[1] if len(sys.argv) > 1 else "gaussian"
n, w, h = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000, 1920, 1080
dev = torch.device("cuda", 0)
ctx = d.Context(0); st = torch.cuda.Stream(dev); torch.cuda.set_stream(st); ctx.use_torch_stream()
k, psi = d.kernel_preset(name), d.default_psi(name)
truth = syn.scene_b(n, 1); init = syn.perturb(truth, 2)
cam = syn.orbit_camera(0, 1, w, h, 1600.0)
lrs = torch.from_numpy(syn.learning_rates(init).reshape(-1)).to(dev)
target = torch.empty((h, w, 3), device=dev)
ctx.evaluate_view(k, psi, torch.from_numpy(truth).to(dev), cam, (0, 0, 0), grad_image=torch.zeros_like(target), image_out=target)
p = torch.from_numpy(init).to(dev); g = torch.zeros_like(p); m = torch.zeros(14 * n, device=dev); v = torch.zeros(14 * n, device=dev)
ctx.set_stage_timing(True)
for it in range(4):
    g.zero_()
    loss = ctx.evaluate_view(k, psi, p, cam, (0, 0, 0), target=target, lam=0.2, param_grads=g)
    t = ctx.stage_times()
    ctx.adam_step(p.view(-1), g.view(-1), m, v, lrs, it + 1)
    t["adam"] = ctx.stage_times()["adam"]
    print(it, loss[0], {a: round(b, 3) for a, b in t.items()})
