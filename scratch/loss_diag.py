import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_loss import smooth_pair
import paper_2501_12369_b200 as darbs
from oracle import cpu
port = cpu.load("port")
ctx = darbs.Context(0)
w, h = int(sys.argv[1]), int(sys.argv[2])
x, y = smooth_pair(w, h, seed=7, noise=0.03)
for lam in (0.2, 1.0):
    vals, grad = ctx.loss_total(x, y, lam)
    st, rv, rg = port.loss_total(x.astype(np.float64), y.astype(np.float64), lam)
    err = np.abs(grad - rg)
    gmax = np.abs(rg).max()
    print("lam", lam, "vals", vals[:3], rv, "gmax", gmax, "max abs err / gmax", err.max() / gmax)
    idx = np.argsort(err.reshape(-1))[::-1][:12]
    for i in idx:
        yy, xx, c = np.unravel_index(i, err.shape)
        print("  y", yy, "x", xx, "c", c, "ref", rg[yy, xx, c] / gmax, "got", grad[yy, xx, c] / gmax, "x", x[yy, xx, c], "y", y[yy, xx, c])
    print("  err percentiles / gmax:", [float(np.percentile(err, p) / gmax) for p in (50, 90, 99, 99.9, 99.99)])
