"""Where does the parameter-gradient error of test_evaluate_view_matches_oracle_chain come from?
Splits it into (a) render backward (splat gradients) and (b) the FP32 preprocess-backward chain."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2501_12369_b200 as darbs  # noqa: E402
from oracle import cpu  # noqa: E402
from oracle.cpu import Scene  # noqa: E402
from test_gpu_geometry import DEMO_CAMERA, random_raw  # noqa: E402

port = cpu.load("port")
f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731


def rel(a, b, floor):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)


for name in sys.argv[1:] or ["raised-cosine"]:
    k, gk, psi = port.preset(name), darbs.kernel_preset(name), port.default_psi(name)
    n, w, h = 600, 64, 64
    raw = random_raw(n, 9, scale_lo=0.02, scale_hi=0.08, spread=0.9)
    gimg = f32(port.random_image_grad(w, h, 77))
    with darbs.Context(0) as ctx:
        pg = np.zeros((n, 14), np.float32)
        ctx.evaluate_view(gk, psi, raw, DEMO_CAMERA, (0, 0, 0), grad_image=gimg, param_grads=pg)
        sg_gpu = ctx.backward(gk, gimg, n)
    prims = port.realize(raw.astype(np.float64))
    st, pr = port.project(k, psi, prims, DEMO_CAMERA)
    vis = np.flatnonzero(pr["valid"])
    s = Scene(pr["mu2"][vis], None, pr["conic"][vis], pr["radius"][vis], pr["depth"][vis], prims[vis, 10],
              prims[vis, 11:14])
    fr = port.forward(k, s, w, h, (0, 0, 0), threads=0, keep=True)
    st, sg = port.backward(fr["handle"], k, gimg.astype(np.float64), s, threads=0)
    port.forward_free(fr["handle"])
    ref = port.param_grads(psi, vis.astype(np.int32), sg, s.conic, s.opacity, s.rgb, prims, DEMO_CAMERA)
    floor = 1e-4 * max(1.0, np.abs(ref).max())
    e = rel(pg, ref, floor)
    i, j = np.unravel_index(e.argmax(), e.shape)
    print(name, "end-to-end", e.max(), (i, j), pg[i, j], ref[i, j], "floor", floor)
    # (a) GPU splat grads through the ORACLE chain
    sgg = np.asarray(sg_gpu, np.float64)[vis]
    mid = port.param_grads(psi, vis.astype(np.int32), sgg, s.conic, s.opacity, s.rgb, prims, DEMO_CAMERA)
    e2 = rel(mid, ref, floor)
    print("  render_bwd share (GPU splat grads, FP64 chain):", e2.max(), np.unravel_index(e2.argmax(), e2.shape),
          "at worst elem:", e2[i, j])
    e3 = rel(pg, mid, floor)
    print("  FP32 chain share (GPU chain vs FP64 chain on the same splat grads):", e3.max(), "at worst elem:", e3[i, j])
    print("  splat grads of prim", i, "gpu", sg_gpu[i], "ref", sg[np.searchsorted(vis, i)])
    print("  params", raw[i])
