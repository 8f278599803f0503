import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2501_12369_b200 as darbs
from oracle import cpu
import test_gpu_loss as L
from conftest import f32
port, ctx = cpu.load("port"), darbs.Context(0)
seed = int(sys.argv[1])
rng = np.random.default_rng(seed)
w, h = int(rng.integers(1, 150)), int(rng.integers(1, 120))
lam = float(rng.choice([0.0, 0.2, 1.0, float(np.round(rng.uniform(0, 1), 3))]))
mode = int(rng.integers(0, 3))
if mode == 0:
    x, y = f32(rng.uniform(0, 1, (h, w, 3))), f32(rng.uniform(0, 1, (h, w, 3)))
elif mode == 1:
    x, y = L.smooth_pair(w, h, int(rng.integers(0, 1000)), noise=float(rng.choice([0.005, 0.02, 0.1])))
else:
    x = L.smooth_pair(w, h, int(rng.integers(0, 1000)))[0]
    y = f32(x + rng.normal(scale=1e-4, size=x.shape))
print(w, h, lam, mode)
vals, grad = ctx.loss_total(x, y, lam)
st, ref_vals, ref_grad = port.loss_total(x.astype(np.float64), y.astype(np.float64), lam)
print("vals", vals, "ref", ref_vals)
d = x.astype(np.float64) - y
print("mse", vals[3], (d * d).mean())
print("grad max err", np.abs(grad - ref_grad).max(), "of", np.abs(ref_grad).max(), "n differing sign", int((np.sign(grad) != np.sign(ref_grad)).sum()))
print("exact ties d == 0:", int((d == 0).sum()))
