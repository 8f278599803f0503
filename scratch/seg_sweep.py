"""cull + render_fwd time against the cull segment (darbs_cuda_set_cull_segment), per DARBF kernel."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_12369_b200 as darbs
from paper_2501_12369_b200 import synthetic as syn

n = int(sys.argv[1]); w, h = int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda", 0)
ctx = darbs.Context(0); ctx.use_torch_stream()
truth = syn.scene_b(n, 1); init = syn.perturb(truth, 2)
cam = syn.orbit_camera(0, 1, w, h, 1600.0 * w / 1920)
truth_d = torch.from_numpy(truth).to(dev); p = torch.from_numpy(init).to(dev); g = torch.zeros((n, 14), device=dev)
for name in ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"]:
    k, psi = darbs.kernel_preset(name), darbs.default_psi(name)
    target = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    ctx.set_cull_segment(1 << 30)
    ctx.evaluate_view(k, psi, truth_d, cam, (0, 0, 0), grad_image=torch.zeros_like(target), image_out=target)
    row = []
    for seg in (128, 192, 256, 384, 512, 768, 1024, 1 << 30):
        ctx.set_cull_segment(seg)
        for _ in range(2):
            ctx.evaluate_view(k, psi, p, cam, (0, 0, 0), target=target, lam=0.2, param_grads=g, accumulate=False)
        ctx.set_stage_timing(True)
        acc = np.zeros(3)
        for _ in range(5):
            ctx.evaluate_view(k, psi, p, cam, (0, 0, 0), target=target, lam=0.2, param_grads=g, accumulate=False)
            st = ctx.stage_times()
            acc += [st["cull"], st["render_fwd"], st["render_bwd"]]
        ctx.set_stage_timing(False)
        acc /= 5
        row.append(f"{seg if seg < 1 << 30 else 'all'}: {1e3 * acc[0]:.0f}+{1e3 * acc[1]:.0f}={1e3 * (acc[0] + acc[1]):.0f} (bwd {1e3 * acc[2]:.0f})")
    print(name, " | ".join(row), flush=True)
