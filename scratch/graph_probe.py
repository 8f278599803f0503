"""Is an iteration capturable in a CUDA graph in the entry-capacity mode, and what does a replay cost?"""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_12369_b200 as d
from paper_2501_12369_b200 import synthetic as syn

n, w, h = 1_000_000, 1920, 1080
dev = torch.device("cuda", 0)
ctx = d.Context(0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
ctx.use_torch_stream()
name = sys.argv[1] if len(sys.argv) > 1 else "gaussian"
k, psi = d.kernel_preset(name), d.default_psi(name)
truth = syn.scene_b(n, 1); init = syn.perturb(truth, 2)
cam = syn.orbit_camera(0, 1, w, h, 1600.0)
target = torch.empty((h, w, 3), device=dev)
ctx.evaluate_view(k, psi, torch.from_numpy(truth).to(dev), cam, (0, 0, 0), grad_image=torch.zeros_like(target), image_out=target)
p = torch.from_numpy(init).to(dev); g = torch.zeros_like(p)
m = torch.zeros(14 * n, device=dev); v = torch.zeros(14 * n, device=dev)
lrs = torch.from_numpy(syn.learning_rates(init).reshape(-1)).to(dev)

def it(t):
    ctx.evaluate_view(k, psi, p, cam, (0, 0, 0), target=target, lam=0.2, param_grads=g, want_loss=False, accumulate=False)
    ctx.adam_step(p.view(-1), g.view(-1), m, v, lrs, t)

for t in range(1, 4): it(t)
wc = ctx.work_counters()
ctx.set_entry_capacity(int(wc["entries"] * 1.25))
for t in range(4, 7): it(t)
torch.cuda.synchronize()
def timed(fn, reps=30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn(i) for i in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
print("eager, capacity mode: %.1f us / iteration" % timed(lambda i: it(7 + i)))
graph = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(graph, stream=st):
        ctx.use_torch_stream()
        ctx.evaluate_view(k, psi, p, cam, (0, 0, 0), target=target, lam=0.2, param_grads=g, want_loss=False, accumulate=False)
    print("captured evaluate_view")
    def rep(i):
        graph.replay()
        ctx.adam_step(p.view(-1), g.view(-1), m, v, lrs, 40 + i)
    print("graph replay + eager adam: %.1f us / iteration" % timed(rep))
except Exception as e:
    print("capture failed:", repr(e)[:500])
