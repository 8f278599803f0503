"""Where do the 3-4 % between the device-resident and the end-to-end iteration go?  Variants of one
training iteration (gaussian, 1 M, 1080p): target resident / prefetched from pinned host memory,
loss not read / read one iteration late."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_12369_b200 as d
from paper_2501_12369_b200 import synthetic as syn

n, w, h = 1_000_000, 1920, 1080
dev = torch.device("cuda", 0)
ctx = d.Context(0); st = torch.cuda.Stream(dev); torch.cuda.set_stream(st); ctx.use_torch_stream()
name = "gaussian"
k, psi = d.kernel_preset(name), d.default_psi(name)
truth = syn.scene_b(n, 1); init = syn.perturb(truth, 2)
cam = syn.orbit_camera(0, 1, w, h, 1600.0)
target = torch.empty((h, w, 3), device=dev)
ctx.evaluate_view(k, psi, torch.from_numpy(truth).to(dev), cam, (0, 0, 0), grad_image=torch.zeros_like(target), image_out=target)
hosts = [torch.empty((h, w, 3), pin_memory=True) for _ in range(2)]
for t_ in hosts: t_.copy_(target.cpu())
hosts_np = [t_.numpy() for t_ in hosts]
p = torch.from_numpy(init).to(dev); g = torch.zeros_like(p)
m = torch.zeros(14 * n, device=dev); v = torch.zeros(14 * n, device=dev)
lrs = torch.from_numpy(syn.learning_rates(init).reshape(-1)).to(dev)
tcount = [0]

def run(host_target, read_loss, reps=40):
    pend = 0
    def it(i):
        nonlocal pend
        tcount[0] += 1
        tgt = hosts_np[i % 2] if host_target else target
        ctx.evaluate_view(k, psi, p, cam, (0, 0, 0), target=tgt, lam=0.2, param_grads=g, want_loss=False, accumulate=False)
        if host_target:
            ctx.prefetch_target(hosts_np[(i + 1) % 2])
        ctx.adam_step(p.view(-1), g.view(-1), m, v, lrs, tcount[0])
        pend += 1
        if read_loss and pend > 1:
            ctx.pop_loss(); pend -= 1
    for i in range(4): it(i)
    while pend and read_loss: ctx.pop_loss(); pend -= 1
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps): it(i)
    while pend and read_loss: ctx.pop_loss(); pend -= 1
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3

for rep in range(2):
    for ht in (False, True):
        for rl in (False, True):
            print(f"host target {ht!s:5} read loss {rl!s:5}: {run(ht, rl):7.1f} us / iteration", flush=True)
