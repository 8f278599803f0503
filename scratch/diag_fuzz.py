"""Replay one chain seed of tests/fuzz_cases.py and split the worst parameter-gradient error:
render backward (splat gradients on the oracle's float32 splats) vs the preprocess backward."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2501_12369_b200 as darbs
from oracle import cpu
from oracle.cpu import Scene
import fuzz_cases as F
from conftest import f32, rel_err, scene_f32

seed = int(sys.argv[1])
port, ctx = cpu.load("port"), darbs.Context(0)
c = F.chain_case(port, darbs, seed)
rng, name, psi, w, h, cam, n, raw, lam, use_loss = (c[key] for key in ("rng", "name", "psi", "w", "h", "cam", "n", "raw", "lam", "use_loss"))
k, gk = port.preset(name), darbs.kernel_preset(name)
print(c["log"])
r32 = lambda a: a.astype(np.float32).astype(np.float64)
prims = port.realize(raw.astype(np.float64))
st, pr = port.project(k, psi, prims, cam)
vis = np.flatnonzero(pr["valid"]).astype(np.int32)
s = Scene(r32(pr["mu2"][vis]), None, r32(pr["conic"][vis]), pr["radius"][vis], r32(pr["depth"][vis]),
          r32(prims[vis, 10]), r32(prims[vis, 11:14]))
fr = port.forward(k, s, w, h, (0, 0, 0), threads=0, keep=True)
img = np.zeros((h, w, 3), np.float32); zero = np.zeros_like(img)
pg = np.zeros((n, 14), np.float32)
if use_loss:
    ctx.evaluate_view(gk, psi, raw, cam, (0, 0, 0), grad_image=zero, image_out=img)
    target = f32(img + rng.choice([-1.0, 1.0], img.shape) * rng.uniform(0.02, 0.15, img.shape))
    vals = ctx.evaluate_view(gk, psi, raw, cam, (0, 0, 0), target=target, lam=lam, param_grads=pg)
    st, ref_vals, gimg = port.loss_total(fr["image"], target.astype(np.float64), lam)
    # the GPU's own dL/dimage for the same images
    st, _, gimg_gpuimg = port.loss_total(img.astype(np.float64), target.astype(np.float64), lam)
    print("loss", vals, ref_vals, "max |gimg(oracle img) - gimg(gpu img)|", np.abs(gimg - gimg_gpuimg).max(), "of", np.abs(gimg).max())
else:
    gimg = r32(port.random_image_grad(w, h, int(rng.integers(0, 100))))
    ctx.evaluate_view(gk, psi, raw, cam, (0, 0, 0), grad_image=f32(gimg), param_grads=pg, image_out=img)
st, sg = port.backward(fr["handle"], k, gimg, s, threads=0)
ref = port.param_grads(psi, vis, sg, s.conic, s.opacity, s.rgb, prims, cam)
floor = np.maximum(1e-3 * np.abs(ref).max(axis=0, keepdims=True), 1e-12)
err = rel_err(pg, ref, floor)
i, c = np.unravel_index(err.argmax(), err.shape)
print("worst", err.max(), "prim", i, "col", c, "gpu", pg[i, c], "ref", ref[i, c], "col max", np.abs(ref[:, c]).max())
print("n bad", int((err > 2e-3).sum()), "cols", np.unique(np.nonzero(err > 2e-3)[1]))
j = int(np.flatnonzero(vis == i)[0])
print("splat: mu", s.mu2[j], "conic", s.conic[j], "radius", s.radius[j], "depth", s.depth[j], "opacity", s.opacity[j])
a, b2, c2 = s.conic[j]
ev = np.linalg.eigvalsh(np.array([[a, b2], [b2, c2]]))
print("conic eigen", ev, "kappa", ev[1] / ev[0])
# render backward alone on the same float32 splats and the same dL/dimage
ctx.forward(gk, **scene_f32(s), width=w, height=h, background=(0, 0, 0))
got_sg = ctx.backward(gk, f32(gimg), s.n)
se = rel_err(got_sg, sg, np.maximum(1e-3 * np.abs(sg).max(axis=0, keepdims=True), 1e-12))
print("splat grads of that splat gpu", got_sg[j]); print("                      ref", sg[j])
print("splat-grad worst err overall", se.max(), "at", np.unravel_index(se.argmax(), se.shape), "this splat", se[j])
# preprocess backward alone: oracle's splat grads through the GPU's FP32 chain is not exposed; use FP64 ABI
print("row gpu", pg[i]); print("row ref", ref[i])
# which stage carries the error: the oracle's FP64 preprocess-backward fed the GPU's splat gradients
ref2 = port.param_grads(psi, vis, got_sg.astype(np.float64), s.conic, s.opacity, s.rgb, prims, cam)
print("FP64 chain on GPU splat grads vs ref:", rel_err(ref2, ref, floor).max(), " | GPU chain vs FP64 chain on GPU splat grads:", rel_err(pg, ref2, floor).max())
print("elementwise abs err / colmax:", (np.abs(pg[i] - ref[i]) / np.abs(ref).max(axis=0)))
x = float(raw[i, 10])
o64 = 1.0 / (1.0 + np.exp(-x))
print("raw logit", x, "sigmoid f64", o64, "oracle prims[10]", prims[i, 10], "gpu realize", float(ctx.realize(raw)[i, 10]), "splat opacity", s.opacity[j])
print("d_opacity gpu", got_sg[j, 3], "ref", sg[j, 3], " ref*o(1-o)", sg[j, 3] * o64 * (1 - o64), "pg col10 gpu", pg[i, 10], "ref", ref[i, 10])
# the render backward on the GPU's OWN projected splats (what evaluate_view rasterizes)
gp = ctx.project(gk, psi, ctx.realize(raw), cam)
vv = gp["valid"] == 1
prg = ctx.realize(raw)
own = dict(mu2=gp["mu2"][vv], conic=gp["conic"][vv], radius=gp["radius"][vv], depth=gp["depth"][vv], opacity=prg[vv, 10], rgb=np.ascontiguousarray(prg[vv, 11:14]))
o1 = ctx.forward(gk, **own, width=w, height=h, background=(0, 0, 0))
sg_own = ctx.backward(gk, f32(gimg), int(vv.sum()))
print("d_opacity on own splats", sg_own[j, 3], "on oracle-rounded splats", got_sg[j, 3], "implied by pg", pg[i, 10] / (o64 * (1 - o64)))
for key in ("mu2", "conic", "depth", "opacity"):
    a_, b_ = own[key][j], getattr(s, key)[j]
    print(key, "own", a_, "oracle f32", f32(b_), "equal" if np.array_equal(f32(a_), f32(b_)) else "DIFFERENT")
o2 = ctx.forward(gk, **scene_f32(s), width=w, height=h, background=(0, 0, 0))
print("processed differ at", int((o1["processed"] != o2["processed"]).sum()), "contributors differ at", int((o1["contributors"] != o2["contributors"]).sum()), "max image diff", np.abs(o1["image"] - o2["image"]).max())
sys.path.insert(0, os.path.join(ROOT, "scratch"))
import emu_chain
print("---- numpy emulation of the chain for prim", i)
emu_chain.compare(raw[i].astype(np.float64), cam, psi, got_sg[j].astype(np.float64))
