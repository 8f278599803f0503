"""Runs forward+backward of one DARBF kernel at 1M splats 1080p (input A) a few times: the
command ncu wraps for the per-kernel captures under profiles/."""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2501_12369_b200 as d
from oracle import cpu
name = sys.argv[1] if len(sys.argv) > 1 else "gaussian"
n, w, h = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000, 1920, 1080
port = cpu.load("port"); k = port.preset(name)
s = port.random_scene(k, n, w, h, 0)
f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
import torch
dev = torch.device("cuda", 0)
T = lambda a: torch.from_numpy(f32(a)).to(dev)
mu2, conic, radius, depth, opacity, rgb = map(T, (s.mu2, s.conic, s.radius, s.depth, s.opacity, s.rgb))
g = torch.randn((h, w, 3), device=dev)
ctx = d.Context(0); gk = d.kernel_preset(name)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st); ctx.use_torch_stream()
ctx.set_stage_timing(True)
for it in range(4):
    out = ctx.forward(gk, mu2, conic, radius, depth, opacity, rgb, w, h, (0.1, 0.2, 0.3), aux=False)
    t1 = ctx.stage_times()
    grads = ctx.backward(gk, g, n)
    t2 = ctx.stage_times()
    print(it, "fwd", t1["binning"], t1["render_fwd"], "bwd", t2["render_bwd"])
print(ctx.work_counters())
