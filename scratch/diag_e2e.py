import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2501_12369_b200 as d
from paper_2501_12369_b200 import synthetic as syn
name = sys.argv[1] if len(sys.argv) > 1 else "half-cosine-sq"
n, w, h = 1000000, 1920, 1080
dev = torch.device("cuda", 0)
ctx = d.Context(0); st = torch.cuda.Stream(dev); torch.cuda.set_stream(st); ctx.use_torch_stream()
k, psi = d.kernel_preset(name), d.default_psi(name)
truth = syn.scene_b(n, 1); init = syn.perturb(truth, 2)
cam = syn.orbit_camera(0, 1, w, h, 1600.0)
lrs = torch.from_numpy(syn.learning_rates(init).reshape(-1)).to(dev)
target = torch.empty((h, w, 3), device=dev)
ctx.evaluate_view(k, psi, torch.from_numpy(truth).to(dev), cam, (0, 0, 0), grad_image=torch.zeros_like(target), image_out=target)
host = target.cpu().pin_memory(); hnp = host.numpy()
p = torch.from_numpy(init).to(dev); g = torch.zeros_like(p); m = torch.zeros(14 * n, device=dev); v = torch.zeros(14 * n, device=dev)
def run(mode, iters=20, timing=False):
    ctx.set_stage_timing(timing)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    acc = {}
    for it in range(iters):
        g.zero_()
        tgt = hnp if mode == "host" else target
        ctx.evaluate_view(k, psi, p, cam, (0, 0, 0), target=tgt, lam=0.0, param_grads=g, want_loss=False)
        if mode == "host": ctx.prefetch_target(hnp)
        if timing:
            t = ctx.stage_times()
            for a, b in t.items(): acc[a] = acc.get(a, 0) + b / iters
        ctx.adam_step(p.view(-1), g.view(-1), m, v, lrs, it + 1)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / iters
    print(mode, "timing" if timing else "free", f"{dt*1e3:.3f} ms/iter", {a: round(b, 3) for a, b in acc.items()})
for mode in ("device", "host", "device", "host"):
    run(mode)
run("device", timing=True); run("host", timing=True)
# raw copy speed
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
buf = torch.empty_like(target)
e0.record(); buf.copy_(host, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("H2D 24.9 MB:", e0.elapsed_time(e1), "ms")
