"""Exploration behind tests/test_gpu_full_size.py::test_training_chain_*: error statistics of the
1 M-primitive scene-B training iteration (evaluate_view + Adam) against the oracle chain."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_12369_b200 as darbs
from paper_2501_12369_b200 import synthetic as syn
from oracle import cpu

N, W, H = int(os.environ.get("N", 1_000_000)), 1920, 1080
ITERS = int(os.environ.get("ITERS", 2))
port = cpu.load("port")
ctx = darbs.Context(0)
truth = syn.scene_b(N, 1)
init = syn.perturb(truth, 2)
lrs = syn.learning_rates(init).reshape(-1)
cam = syn.orbit_camera(0, 1, W, H, 1600.0)
for name in sys.argv[1:] or ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"]:
    k, gk, psi = port.preset(name), darbs.kernel_preset(name), port.default_psi(name)
    target = np.zeros((H, W, 3), np.float32)
    ctx.evaluate_view(gk, psi, truth, cam, (0, 0, 0), grad_image=np.zeros_like(target), image_out=target)
    p_gpu = init.copy(); m_gpu = np.zeros(14 * N, np.float32); v_gpu = np.zeros(14 * N, np.float32)
    p_ref = init.astype(np.float64); m_ref = np.zeros(14 * N); v_ref = np.zeros(14 * N)
    for it in range(1, ITERS + 1):
        pg = np.zeros((N, 14), np.float32)
        loss = ctx.evaluate_view(gk, psi, p_gpu, cam, (0, 0, 0), target=target, lam=0.2, param_grads=pg)
        t0 = time.time()
        prims = port.realize(p_ref)
        st, pr = port.project(k, psi, prims, cam)
        vis = np.flatnonzero(pr["valid"]).astype(np.int32)
        f = lambda a: a.astype(np.float32).astype(np.float64)
        s = cpu.Scene(f(pr["mu2"][vis]), None, f(pr["conic"][vis]), f(pr["radius"][vis]), f(pr["depth"][vis]),
                      f(prims[vis, 10]), f(prims[vis, 11:14]))
        fr = port.forward(k, s, W, H, (0, 0, 0), threads=0, keep=True)
        st, vals, gimg = port.loss_total(fr["image"], target.astype(np.float64), 0.2)
        st, sg = port.backward(fr["handle"], k, gimg, s, threads=0)
        port.forward_free(fr["handle"])
        ref = port.param_grads(psi, vis, sg, s.conic, s.opacity, s.rgb, prims, cam)
        print(f"{name} it {it}: oracle {time.time()-t0:.1f}s loss gpu {loss[0]:.9f} ref {vals[0]:.9f} rel {abs(loss[0]-vals[0])/vals[0]:.2e}")
        a, b = pg.astype(np.float64), ref
        colmax = np.abs(b).max(axis=0)
        for floor_name, floor in (("1e-4", 1e-4), ("1e-3*colmax", 1e-3 * colmax[None, :]), ("1e-4*colmax", 1e-4 * colmax[None, :])):
            err = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
            print(f"   floor {floor_name}: max {err.max():.3e} p99.99 {np.quantile(err, 0.9999):.3e} frac>1e-3 {(err>1e-3).mean():.3e} worst col {err.max(axis=0).argmax()}")
        print("   colmax", np.array2string(colmax, precision=3))
        if it == 1:
            # leg B alone: the oracle's own dL/dimage (rounded to float32) drives the GPU's backward chain
            pg2 = np.zeros((N, 14), np.float32)
            g32 = gimg.astype(np.float32)
            ctx.evaluate_view(gk, psi, p_gpu, cam, (0, 0, 0), grad_image=g32, param_grads=pg2)
            fr2 = port.forward(k, s, W, H, (0, 0, 0), threads=0, keep=True)
            st, sg2 = port.backward(fr2["handle"], k, g32.astype(np.float64), s, threads=0)
            port.forward_free(fr2["handle"])
            ref2 = port.param_grads(psi, vis, sg2, s.conic, s.opacity, s.rgb, prims, cam)
            a2 = pg2.astype(np.float64)
            cm2 = np.abs(ref2).max(axis=0)
            for floor_name, floor in (("1e-3*colmax", 1e-3 * cm2[None, :]), ("1e-4*colmax", 1e-4 * cm2[None, :])):
                err = np.abs(a2 - ref2) / np.maximum(np.maximum(np.abs(a2), np.abs(ref2)), floor)
                print(f"   [given dL/dimage] floor {floor_name}: max {err.max():.3e} p99.99 {np.quantile(err, 0.9999):.3e} p99.9999 {np.quantile(err, 0.999999):.3e} frac>1e-3 {(err>1e-3).mean():.3e} worst col {err.max(axis=0).argmax()}")
            gl = np.zeros((H, W, 3), np.float32)
            (lt, grad_gpu) = ctx.loss_total(fr["image"].astype(np.float32), target, 0.2)
            dg = np.abs(grad_gpu.astype(np.float64) - gimg)
            print(f"   loss grad: max |dg| {dg.max():.3e} of max |g| {np.abs(gimg).max():.3e}; elements off by > 1e-8: {(dg > 1e-8).sum()}")
        # Adam on each side's own gradients; then compare parameters where the step is decided
        ctx.adam_step(p_gpu.reshape(-1), pg.reshape(-1), m_gpu, v_gpu, lrs, it)
        st, p_new, m_ref, v_ref = port.adam_step(p_ref.reshape(-1), ref.reshape(-1), m_ref, v_ref, lrs.astype(np.float64), it)
        p_ref = p_new.reshape(N, 14)
        d = np.abs(p_gpu.astype(np.float64) - p_ref) / lrs.reshape(N, 14)
        print(f"   params: max |dp|/lr {d.max():.3e}, frac > 1e-2 {(d > 1e-2).mean():.3e}, > 1e-3 {(d>1e-3).mean():.3e}")
