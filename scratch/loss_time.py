"""Times darbs_cuda_loss_total at 1920x1080 on device arrays (CUDA events through stage timing)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_12369_b200 as darbs

ctx = darbs.Context(0)
ctx.use_torch_stream()
x = torch.rand((1080, 1920, 3), device="cuda")
y = (x + 0.02 * torch.randn_like(x)).clamp(0, 1)
ctx.set_stage_timing(True)
for lam in (0.0, 0.2):
    for _ in range(3):
        ctx.loss_total(x, y, lam)
    ts = []
    for _ in range(10):
        ctx.loss_total(x, y, lam)
        ts.append(ctx.stage_times()["loss"])
    print(f"lambda={lam}: loss stage {min(ts)*1e3:.1f} us (min of 10), median {sorted(ts)[5]*1e3:.1f} us")
