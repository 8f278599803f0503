#!/usr/bin/env python
"""bench.py — the reference's headline workload on the B200-native rasterizer.

Workload (BASELINE.json configs[2], the configuration the metric "train iters/sec (fwd+bwd) at
1M splats 1080p per DARBF kernel" is quoted on): 1 000 000 synthetic primitives, 1920x1080, one
camera view per GPU, one full training iteration per DARBF kernel = preprocess -> bin/sort ->
render forward -> loss (L1 + D-SSIM, lambda 0.2) -> render backward -> preprocess backward -> Adam
(fit_scene's evaluate + adam_step, src/fit3d.cpp:104-184).  One "step" runs that iteration once
for each of the four kernels (gaussian, half-cosine-sq, raised-cosine, inv-multiquadratic);
``value`` = view-iterations per second over the whole job (4 * steps * n_gpus / seconds), i.e. the
harmonic mean over the four kernels; per-kernel numbers are in ``per_kernel``.

  python bench.py [--gpus N] [--steps K] [--warmup W]            (torchrun for N > 1)
  N > 1 (or --config 3) runs BASELINE.json configs[3] instead: 3 M primitives, 64 cameras sharded by
  view over the GPUs, one NCCL all-reduce of the gradients per iteration (run_config3).
  python bench.py --impl reference ...   times the reference's own CPU code (oracle/_ref) on the
                                         host cores on the same workload at full size (repetitions capped).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

KERNELS = ["gaussian", "half-cosine-sq", "raised-cosine", "inv-multiquadratic"]
# algorithmic flops / MUFU ops per visit and per contributor, SURVEY.md §8d
F_K = {"gaussian": (1, 1), "half-cosine-sq": (3, 1), "raised-cosine": (5, 2), "inv-multiquadratic": (2, 1)}
FP_K = {"gaussian": (1, 0), "half-cosine-sq": (2, 1), "raised-cosine": (4, 2), "inv-multiquadratic": (3, 0)}
METRIC = "train_view_iters_per_sec_1M_splats_1080p"
UNIT = "view-iters/s (fwd+bwd+Adam, mean over the 4 DARBF kernels)"
SAMPLE_FRACTION = 16
LAMBDA = 0.2  # FitConfig::lambda, include/darbs/fit_common.hpp:16: L = (1 - lambda) L1 + lambda (1 - SSIM)/2


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=None, choices=[2, 3],
                    help="BASELINE.json configs[] index: 2 = 1M splats, one view per GPU (default at --gpus 1); "
                         "3 = 3M splats, 64 cameras sharded by view, one gradient all-reduce per iteration "
                         "(default at --gpus > 1)")
    ap.add_argument("--views", type=int, default=64, help="cameras of configs[3]")
    ap.add_argument("--no-single-gpu-ref", action="store_true",
                    help="configs[3], N > 1: skip rank 0's single-GPU pass over all views of the same workload")
    ap.add_argument("--splats", type=int, default=None)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--focal", type=float, default=1600.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--table", action="store_true",
                    help="with --impl reference: time the reference's CPU code on BASELINE.json configs[0] and "
                         "configs[1] too (the rows of BASELINE.md section 4) instead of the headline workload")
    ap.add_argument("--exact", type=int, default=1, help="FP64 guard-band re-decisions (default on)")
    ap.add_argument("--entry-capacity", default="0",
                    help="0 (default): every view waits (an event) for its tile-entry count K; auto: after the warm-up "
                         "the context is promised 1.25 x the K of each kernel's view (darbs_cuda_set_entry_capacity), as a "
                         "training loop would from its previous iterations, and no iteration waits for K.  Measured: "
                         "810 view-iterations/s with auto against 824 with the wait (the GPU is never starved by it; the "
                         "capacity-sized grids and clears cost a little)")
    ap.add_argument("--no-cuda-graph", action="store_true",
                    help="device-resident arm of the single-GPU workload: by default each kernel's view is captured once "
                         "into a CUDA graph and replayed (possible because a promised entry capacity leaves no host "
                         "synchronisation in a view; Adam stays an eager launch: its bias correction changes every step).  "
                         "Measured: 856 view-iterations/s replayed against 825 launched eagerly.  The end-to-end arm "
                         "always launches eagerly (its target uploads run on a second stream)")
    args = ap.parse_args()
    args.cuda_graph = not args.no_cuda_graph
    if args.config is None:
        args.config = 2 if args.gpus == 1 else 3
    if args.splats is None:
        args.splats = 1_000_000 if args.config == 2 else 3_000_000
    return args


# ------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
                pw.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        # "under load": samples in the upper half of the power draw seen
        thr = 0.5 * (min(pw) + max(pw))
        load = [s for s, p in zip(sm, pw) if p >= thr] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": float(max(pw))}


# --------------------------------------------------------------------------- CPU reference arm
def cpu_iteration(orc, cpu, name, raw64, cam, target, lrs64, state, threads):
    """fit_scene's evaluate (one view) + adam_step, built from the oracle library's functions
    exactly as src/fit3d.cpp:104-184 sequences them.  Returns seconds."""
    k = orc.preset(name)
    psi = orc.default_psi(name)
    w, h = int(cam[4]), int(cam[5])
    t0 = time.perf_counter()
    prims = orc.realize(raw64)
    st, pr = orc.project(k, psi, prims, cam)
    vis = np.flatnonzero(pr["valid"]).astype(np.int32)
    s = cpu.Scene(pr["mu2"][vis], None, pr["conic"][vis], pr["radius"][vis], pr["depth"][vis], prims[vis, 10],
                  prims[vis, 11:14])
    fr = orc.forward(k, s, w, h, (0.0, 0.0, 0.0), threads=threads, keep=True)
    st, _vals, gimg = orc.loss_total(fr["image"], target, LAMBDA)  # fit3d.cpp:122
    st, sg = orc.backward(fr["handle"], k, gimg, s, threads=threads)
    orc.forward_free(fr["handle"])
    grads = orc.param_grads(psi, vis, sg, s.conic, s.opacity, s.rgb, prims, cam)
    state["t"] += 1
    st, p, m, v = orc.adam_step(raw64.reshape(-1), grads.reshape(-1), state["m"], state["v"], lrs64.reshape(-1),
                                state["t"])
    state["m"], state["v"] = m, v
    raw64[...] = p.reshape(raw64.shape)
    return time.perf_counter() - t0, int(fr["processed"].sum())


def cpu_setup(args, fraction):
    """The CPU checker and the workload (fraction = 1: the GPU arm's own scene, camera and start;
    otherwise a 1/fraction sample at equal splat density).  paper_2501_12369_b200.synthetic is pure
    numpy: importing it does not load the product library (the package loads it lazily)."""
    from oracle import cpu
    from paper_2501_12369_b200 import synthetic as syn

    kind = "reference" if cpu.available("reference") else "port"
    orc = cpu.load(kind)
    if fraction == 1:
        truth = syn.scene_b(args.splats, 1)
        cam = syn.orbit_camera(0, 1, args.width, args.height, args.focal)
    else:
        smp = syn.sample_workload(args.splats, args.width, args.height, args.focal, fraction)
        truth = syn.scene_b(smp["n"], 1, half_extent=smp["half_extent"])
        cam = syn.orbit_camera(0, 1, smp["width"], smp["height"], smp["focal"])
    init = syn.perturb(truth, 2)
    lrs = syn.learning_rates(init)
    return cpu, orc, kind, truth, cam, init, lrs


def cpu_target(orc, cpu, name, truth, cam, threads):
    k = orc.preset(name)
    psi = orc.default_psi(name)
    prims = orc.realize(truth.astype(np.float64))
    st, pr = orc.project(k, psi, prims, cam)
    vis = np.flatnonzero(pr["valid"])
    s = cpu.Scene(pr["mu2"][vis], None, pr["conic"][vis], pr["radius"][vis], pr["depth"][vis], prims[vis, 10],
                  prims[vis, 11:14])
    return orc.forward(k, s, int(cam[4]), int(cam[5]), (0.0, 0.0, 0.0), threads=threads)["image"]


def reference_table(args):
    """The CPU side of BASELINE.md section 4 for the configurations bench.py's headline does not cover:
    configs[0] (10 k random splats, 256 x 256, half-cosine-sq, forward + backward; input A, the reference's
    own random_scene) and configs[1] (1 M splats 1080p forward render per kernel; scene B projected by the
    reference's own project_primitive).  The reference's own sources (oracle/_ref), steady clock around the
    calls, 1 warm-up + 3 repetitions (1 at 1 M splats)."""
    from oracle import cpu
    from paper_2501_12369_b200 import synthetic as syn

    kind = "reference" if cpu.available("reference") else "port"
    orc = cpu.load(kind)
    threads = os.cpu_count() or 1
    out = {"impl": "reference", "kind": kind, "cores": threads}
    k = orc.preset("half-cosine-sq")
    s = orc.random_scene(k, 10_000, 256, 256, 0)
    g = orc.random_image_grad(256, 256, 32)
    rows = {}
    for th in (threads, 1):
        tf = tb = 0.0
        for rep in range(4):
            t0 = time.perf_counter()
            fr = orc.forward(k, s, 256, 256, (0.1, 0.2, 0.3), threads=th, keep=True)
            t1 = time.perf_counter()
            orc.backward(fr["handle"], k, g, s, threads=th)
            t2 = time.perf_counter()
            orc.forward_free(fr["handle"])
            if rep:
                tf += (t1 - t0) / 3
                tb += (t2 - t1) / 3
        rows[f"{th}_threads"] = {"ms_forward": 1e3 * tf, "ms_backward": 1e3 * tb}
    out["config0_10k_256_half-cosine-sq"] = rows
    # the reference's own micro-benchmark sizes (benchmarks/bench.cpp:58-75, 116-117): 200 / 1000 splats, 128 x 128, Gaussian
    kg = orc.preset("gaussian")
    small = {}
    for n_small in (200, 1000):
        sc = orc.random_scene(kg, n_small, 128, 128, 7)
        g1 = np.ones((128, 128, 3))
        tf = tb = 0.0
        for rep in range(12):
            t0 = time.perf_counter()
            fr = orc.forward(kg, sc, 128, 128, (0.1, 0.2, 0.3), threads=1, keep=True)
            t1 = time.perf_counter()
            orc.backward(fr["handle"], kg, g1, sc, threads=1)
            t2 = time.perf_counter()
            orc.forward_free(fr["handle"])
            if rep >= 2:
                tf += (t1 - t0) / 10
                tb += (t2 - t1) / 10
        small[f"{n_small}_splats_128x128_gaussian"] = {"us_forward": 1e6 * tf, "us_backward": 1e6 * tb, "threads": 1}
    out["bm_forward_backward"] = small
    truth = syn.scene_b(args.splats, 1)
    cam = syn.orbit_camera(0, 1, args.width, args.height, args.focal)
    fwd = {}
    for name in ("gaussian", "half-cosine-sq", "raised-cosine"):
        kk, psi = orc.preset(name), orc.default_psi(name)
        t0 = time.perf_counter()
        prims = orc.realize(truth.astype(np.float64))
        st, pr = orc.project(kk, psi, prims, cam)
        vis = np.flatnonzero(pr["valid"])
        sc = cpu.Scene(pr["mu2"][vis], None, pr["conic"][vis], pr["radius"][vis], pr["depth"][vis], prims[vis, 10],
                       prims[vis, 11:14])
        t1 = time.perf_counter()
        orc.forward(kk, sc, args.width, args.height, (0.0, 0.0, 0.0), threads=threads)
        t2 = time.perf_counter()
        fwd[name] = {"ms_preprocess": 1e3 * (t1 - t0), "ms_forward_incl_bin": 1e3 * (t2 - t1), "fps": 1.0 / (t2 - t0)}
    out[f"config1_{args.splats}_splats_{args.width}x{args.height}_forward"] = fwd
    print(json.dumps(out), flush=True)


def run_reference_arm(args):
    """(The reference arm always times configs[2], the configuration the metric is quoted on: a
    full-size configs[3] iteration is 64 views x ~10 s of CPU time.)
    --impl reference: the reference's own CPU implementation (oracle/_ref: its unmodified
    kernel/geometry/rasterizer/loss sources), all host threads, on configs[2] AT FULL SIZE.  One
    full-size iteration is 5-10 s of CPU time, so the arm caps its own repetitions (at most one
    warm-up and two timed iterations per DARBF kernel; DARBS_REF_STEPS / DARBS_REF_WARMUP override)
    and reports the steps it really ran, so that the whole run ends within a few minutes.  The 1/16
    sample the GPU arm's ``cpu_baseline`` leg times is reported beside it as a secondary key."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    steps = max(1, min(args.steps, int(os.environ.get("DARBS_REF_STEPS", "2"))))
    warmup = max(0, min(args.warmup, int(os.environ.get("DARBS_REF_WARMUP", "1"))))
    cpu, orc, kind, truth, cam, init, lrs = cpu_setup(args, fraction=1)
    lrs64 = lrs.astype(np.float64)
    total, per_kernel = 0.0, {}
    for name in KERNELS:
        target = cpu_target(orc, cpu, name, truth, cam, threads)
        raw = init.astype(np.float64).copy()
        state = {"m": np.zeros(raw.size), "v": np.zeros(raw.size), "t": 0}
        for _ in range(warmup):
            cpu_iteration(orc, cpu, name, raw, cam, target, lrs64, state, threads)
        sec = 0.0
        for _ in range(steps):
            dt, _v = cpu_iteration(orc, cpu, name, raw, cam, target, lrs64, state, threads)
            sec += dt
        per_kernel[name] = {"ms_per_iter": 1e3 * sec / steps, "iters_per_s": steps / sec}
        total += sec
        del target, raw, state
    value = len(KERNELS) * steps / total
    sample = (f"the full workload ({args.splats} primitives, {args.width}x{args.height}), {warmup} warm-up + {steps} "
              f"timed full training iterations per kernel ({args.steps} steps / {args.warmup} warm-up requested; "
              f"capped so that the run ends within minutes)")
    # secondary: the bounded 1/16 sample at equal splat density (what the GPU arm's cpu_baseline leg runs)
    secondary = None
    if not args.no_cpu_baseline:
        cb = cpu_baseline(args, single_thread=False)
        secondary = {"value_full_equiv": cb["value"], "sample": cb["sample"]}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warmup, "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": 1e3 * total / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "per_kernel": per_kernel, "sample_1_16": secondary,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n_gpus):
    return {
        "workload": f"{args.splats} synthetic 3-D primitives (scene B, SURVEY 8d), {args.width}x{args.height}, "
                    f"1 orbit view per GPU, full training iteration (preprocess, bin+sort, cull, render fwd, L1 + D-SSIM loss "
                    f"with lambda {LAMBDA}, "
                    f"render bwd, preprocess bwd, Adam) for each of {', '.join(KERNELS)}",
        "splats": args.splats, "width": args.width, "height": args.height, "views_per_step": n_gpus,
        "parallelism": f"view-parallel x{n_gpus}, NCCL all-reduce of 14N f32 parameter gradients" if n_gpus > 1
        else "single GPU",
        "l2_policy": "inputs larger than L2: ~0.5 GB of parameters, Adam state, records and images are "
                     "streamed every iteration (L2 is 126 MB)",
    }


# -------------------------------------------------------------------------------- the GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2501_12369_b200 as darbs
    from paper_2501_12369_b200 import synthetic as syn

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = darbs.Context(local)
    stream = torch.cuda.Stream(dev)  # one stream for torch ops, NCCL hand-off and the library's kernels
    torch.cuda.set_stream(stream)
    ctx.use_torch_stream()
    ctx.set_exact_decisions(bool(args.exact))
    if world > 1:
        ids = [darbs.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        ctx.comm_init(ids[0], rank, world)

    n, w, h = args.splats, args.width, args.height
    truth = syn.scene_b(n, 1)
    init = syn.perturb(truth, 2)
    lrs = torch.from_numpy(syn.learning_rates(init).reshape(-1)).to(dev)
    cam = syn.orbit_camera(rank, max(world, 1), w, h, args.focal)  # view v -> rank v mod G
    truth_d = torch.from_numpy(truth).to(dev)
    bg = (0.0, 0.0, 0.0)  # fit_scene's background, fit3d.cpp:52

    kernels = {name: (darbs.kernel_preset(name), darbs.default_psi(name)) for name in KERNELS}
    state = {}
    for name, (k, psi) in kernels.items():
        target = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
        ctx.evaluate_view(k, psi, truth_d, cam, bg, grad_image=torch.zeros_like(target), image_out=target)
        state[name] = dict(
            params=torch.from_numpy(init).to(dev).clone(), m=torch.zeros(14 * n, device=dev),
            v=torch.zeros(14 * n, device=dev), grads=torch.zeros((n, 14), device=dev), target=target,
            target_host=target.cpu().pin_memory(), t=0)
        state[name]["target_np"] = state[name]["target_host"].numpy()
    torch.cuda.synchronize()

    capacity = {}  # per kernel, filled after the warm-up (--entry-capacity auto)
    graphs, graph_launches, replayed = {}, {}, [0]  # --cuda-graph: one captured view per kernel

    def iteration(name, e2e: bool):
        k, psi = kernels[name]
        s = state[name]
        if capacity:
            ctx.set_entry_capacity(capacity[name])
        # one view per GPU and iteration: the view OVERWRITES the gradient buffer (accumulate=False),
        # which is fit3d.cpp:107's fill followed by the first "+=" without a pass that zeroes 14 N floats
        if e2e:
            # the view's target image comes from pinned host memory through the C ABI
            # (image_space = DARBS_HOST); the loss of every iteration is read back to the host, one
            # iteration late (darbs_cuda_pop_loss) so that the read-back never drains the stream
            loss = ctx.evaluate_view(k, psi, s["params"], cam, bg, target=s["target_np"], lam=LAMBDA,
                                     param_grads=s["grads"], want_loss=False, accumulate=False)
            # the next iteration's target starts its upload under this iteration's render kernels
            ctx.prefetch_target(state[KERNELS[(KERNELS.index(name) + 1) % len(KERNELS)]]["target_np"])
        elif name in graphs:
            loss = None
            graphs[name].replay()
            replayed[0] += graph_launches[name]
        else:
            loss = ctx.evaluate_view(k, psi, s["params"], cam, bg, target=s["target"], lam=LAMBDA,
                                     param_grads=s["grads"], want_loss=False, accumulate=False)
        s["t"] += 1
        if world > 1:  # --config 2 on several GPUs: gradients are summed over the ranks' views, fit3d.cpp:148-158
            ctx.allreduce_adam_step(s["params"].view(-1), s["grads"].view(-1), s["m"], s["v"], lrs, s["t"])
        else:
            ctx.adam_step(s["params"].view(-1), s["grads"].view(-1), s["m"], s["v"], lrs, s["t"])
        if e2e:
            pending[0] += 1
            if pending[0] > 2:  # the loss of two iterations ago: the host stays a full iteration ahead of the read-back
                losses.append(ctx.pop_loss())
                pending[0] -= 1
        return loss

    pending, losses = [0], []

    def drain_losses():
        while pending[0] > 0:
            losses.append(ctx.pop_loss())
            pending[0] -= 1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(steps, e2e):
        """K steps (each = one iteration per kernel), CUDA events on the launching stream."""
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in KERNELS]
              for _ in range(steps)]
        per = {name: 0.0 for name in KERNELS}
        barrier()
        l0 = ctx.launch_count()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record()
        for step in range(steps):  # no synchronisation between steps: the host runs ahead of the GPU
            for (a, b), name in zip(ev[step], KERNELS):
                a.record()
                iteration(name, e2e)
                b.record()
        if e2e:
            drain_losses()  # inside the timed region: every iteration's loss has reached the host
        t_end.record()
        barrier()
        ms = t_start.elapsed_time(t_end)
        for step in range(steps):
            for (a, b), name in zip(ev[step], KERNELS):
                per[name] += a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, per, ctx.launch_count() - l0

    # warm-up (also sizes the workspace), then the device-resident timed region.  nvidia-smi needs
    # a few hundred ms to deliver its first sample, so the sampler runs from the warm-up on.
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    for _ in range(max(args.warmup, 3)):
        for name in KERNELS:
            iteration(name, False)
    if args.entry_capacity == "auto" or args.cuda_graph:
        # what a training loop knows from its previous iterations: K of the kernel's view, plus a quarter
        for name in KERNELS:
            k, psi = kernels[name]
            s = state[name]
            ctx.evaluate_view(k, psi, s["params"], cam, bg, target=s["target"], lam=LAMBDA, param_grads=s["grads"],
                              accumulate=False)
            capacity[name] = int(1.25 * ctx.work_counters()["entries"])
    graph_note = "off (--no-cuda-graph)"
    if args.cuda_graph:
        try:
            for name in KERNELS:
                iteration(name, False)  # buffers and grids sized by the capacity before the capture
            torch.cuda.synchronize()
            for name in KERNELS:
                k, psi = kernels[name]
                s = state[name]
                ctx.set_entry_capacity(capacity[name])
                g = torch.cuda.CUDAGraph()
                l0 = ctx.launch_count()
                with torch.cuda.graph(g, stream=torch.cuda.current_stream()):
                    ctx.use_torch_stream()
                    ctx.evaluate_view(k, psi, s["params"], cam, bg, target=s["target"], lam=LAMBDA,
                                      param_grads=s["grads"], want_loss=False, accumulate=False)
                graphs[name], graph_launches[name] = g, ctx.launch_count() - l0
            graph_note = "one captured view per kernel, replayed; Adam launched eagerly"
        except Exception as e:  # noqa: BLE001 - the eager launches are always available
            graphs.clear()
            graph_note = f"capture failed ({type(e).__name__}); launched eagerly"
            torch.cuda.synchronize()
    ms, per, launches = timed(args.steps, e2e=False)
    launches += replayed[0]
    if graphs:
        # a replayed view cannot report that it outgrew its promised capacity: check K now, eagerly
        ctx.set_entry_capacity(0)
        for name in KERNELS:
            k, psi = kernels[name]
            s = state[name]
            ctx.evaluate_view(k, psi, s["params"], cam, bg, target=s["target"], lam=LAMBDA, accumulate=False)
            if ctx.work_counters()["entries"] > capacity[name]:
                graph_note = f"{name} outgrew its capacity during the timed region; re-timed with eager launches"
        if "outgrew" in graph_note:
            graphs.clear()
            replayed[0] = 0
            if args.entry_capacity != "auto":
                capacity.clear()
            ms, per, launches = timed(args.steps, e2e=False)
    graphs_used, graphs = bool(graphs), {}  # the end-to-end arm below launches eagerly
    capacity_value_arm = dict(capacity)
    if args.entry_capacity != "auto":
        capacity.clear()                    # ... and waits for K as every other caller does by default
    value = len(KERNELS) * args.steps * world / (ms * 1e-3)

    # end-to-end: target image from pinned host memory each iteration, loss read back
    for name in KERNELS:
        iteration(name, True)
    drain_losses()
    losses.clear()
    ms_e2e, per_e2e, _ = timed(args.steps, e2e=True)
    clocks = sampler.stop() if rank == 0 else None
    e2e_value = len(KERNELS) * args.steps * world / (ms_e2e * 1e-3)

    # per-stage device times and work counters (separate, untimed pass with stage events on)
    capacity_used, capacity = dict(capacity), {}
    ctx.set_entry_capacity(0)
    ctx.set_stage_timing(True)
    peaks = ctx.microbench()
    per_kernel = {}
    for name in KERNELS:
        k, psi = kernels[name]
        s = state[name]
        acc = None
        reps = 3
        for _ in range(reps):
            ctx.evaluate_view(k, psi, s["params"], cam, bg, target=s["target"], lam=LAMBDA, param_grads=s["grads"],
                              accumulate=False)
            st = ctx.stage_times()
            ctx.adam_step(s["params"].view(-1), s["grads"].view(-1), s["m"], s["v"], lrs, s["t"] + 1)
            st["adam"] = ctx.stage_times()["adam"]
            acc = st if acc is None else {kk: acc[kk] + st[kk] for kk in st}
        st = {kk: vv / reps for kk, vv in acc.items()}
        wc = ctx.work_counters()
        roof_fwd, roof_bwd = render_rooflines(name, wc, st, peaks)

        per_kernel[name] = {
            "iters_per_s": args.steps * world / (per[name] * 1e-3),
            "iters_per_s_e2e": args.steps * world / (per_e2e[name] * 1e-3),
            "ms_per_iter": per[name] / args.steps,
            "stage_ms": st,
            "render_fps": 1e3 / max(st["preprocess"] + st["binning"] + st["cull"] + st["render_fwd"], 1e-9),
            "work": wc,
            "render_fwd": roof_fwd,
            "render_bwd": roof_bwd,
        }
    ctx.set_stage_timing(False)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # dominant kernel = the render kernel with the largest device time over the four families
    dom = max(((nm, kk) for nm in KERNELS for kk in ("render_fwd", "render_bwd")),
              key=lambda t: per_kernel[t[0]][t[1]]["ms"])
    dk = per_kernel[dom[0]][dom[1]]
    roofline = roofline_record(f"{dom[1]}<{dom[0]}>", dk, peaks)

    hbm_peak = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak = json.load(f).get("hbm_gbs")
    except OSError:
        pass
    if hbm_peak:
        # streaming stages against the measured HBM peak (algorithmic bytes)
        for name in KERNELS:
            st = per_kernel[name]["stage_ms"]
            kk = per_kernel[name]["work"]["entries"]
            per_kernel[name]["hbm_frac"] = {
                # fused preprocess: 56 B of parameters in; 48 B SoA splat, 64 B packed record, 8 B tile
                # rectangle, 4 B tile count, 4 B depth key and 4 B identity order out, per primitive
                "preprocess": (56 + 48 + 64 + 20) * n / (st["preprocess"] * 1e-3) / 1e9 / hbm_peak,
                "preprocess_bwd": (36 + 56 + 56) * n / (st["preprocess_bwd"] * 1e-3) / 1e9 / hbm_peak,
                "adam": 28 * 14 * n / (st["adam"] * 1e-3) / 1e9 / hbm_peak,
                # loss: image + target read twice, three partial maps written and read, gradient written
                "loss": (4 * 12 + 2 * 36 + 12) * w * h / (st["loss"] * 1e-3) / 1e9 / hbm_peak,
                # per splat: depth sort (4 B histogram read + 4 digit passes x 16 B), expand (4 B order + 12 B
                # gathered rectangle and count); per tile entry: 6 B written by expand, tile sort on 16-bit
                # keys (2 passes x 12 B), ranges 2 B
                "binning_sort": (84 * n + 32 * kk) / (st["binning"] * 1e-3) / 1e9 / hbm_peak,
                # cull: 4 B index + 48 B record gather per tile entry (L2-resident records: not HBM)
                # and 48 B written per surviving (block, entry) pair
                "cull": (4 * kk + 48 * per_kernel[name]["work"]["survivors"]) / (st["cull"] * 1e-3) / 1e9 / hbm_peak,
            }

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, world), "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": len(KERNELS) * 12 * w * h,
                "d2h_bytes_per_step": len(KERNELS) * 32,
                "path": "darbs_cuda_evaluate_view with the view's target image in pinned host memory "
                        "(image_space = DARBS_HOST; darbs_cuda_prefetch_target starts each upload on a second "
                        "stream under the previous iteration's render kernels) and every "
                        "iteration's loss read back with darbs_cuda_pop_loss one iteration late; parameters "
                        "stay on the device", "losses_read": len(losses)},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "exact_decisions": bool(args.exact),
        "cuda_graph": {"value_arm": graphs_used, "note": graph_note},
        "entry_capacity": {"value_arm": capacity_value_arm, "e2e_arm": capacity_used,
                           "note": "tile entries promised per kernel (darbs_cuda_set_entry_capacity, 1.25 x the K of the "
                                   "warm-up iterations): what lets a view be captured in a CUDA graph; empty = every view "
                                   "waits (an event) for its K, the library's default and what the end-to-end arm does "
                                   "unless --entry-capacity auto"},
        "per_kernel": per_kernel,
    }
    if world == 1:
        line["e2e_dropin"] = dropin_boundary(ctx, darbs, syn, kernels, truth, cam, w, h)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def render_rooflines(name, wc, st, peaks):
    """algorithmic flops / MUFU ops of the two render kernels from the launch's own
    work counters (V = sum processed, C = sum contributors) against the measured peaks."""
    V, Cn = wc["visits"], wc["contributors"]
    fk, sk = F_K[name]
    fpk, spk = FP_K[name]
    fp32_peak = fp32_peak_of(peaks)
    E = 32 * wc["composited"]  # the stricter count: only the lane-visits the kernels evaluate

    def roof(flops, mufu, ms_k, evaluated):
        t_fp = flops / fp32_peak
        t_mu = mufu / peaks["mufu_per_s"]
        t_ev = max(evaluated[0] / fp32_peak, evaluated[1] / peaks["mufu_per_s"])
        return {"ms": ms_k, "algorithmic_gflop": flops / 1e9, "achieved_tflops": flops / (ms_k * 1e-3) / 1e12,
                "frac_fp32": t_fp / (ms_k * 1e-3), "frac_mufu": t_mu / (ms_k * 1e-3),
                "frac": max(t_fp, t_mu) / (ms_k * 1e-3), "frac_evaluated": t_ev / (ms_k * 1e-3)}

    return (roof(V * (13 + fk) + 9 * Cn, V * sk, st["render_fwd"], (E * (13 + fk) + 9 * Cn, E * sk)),
            roof(V * (13 + fk + fpk) + 57 * Cn, V * (sk + spk) + Cn, st["render_bwd"],
                 (E * (13 + fk + fpk) + 57 * Cn, E * (sk + spk) + Cn)))


def roofline_record(kernel, dk, peaks):
    return {
        "bound": "fp32", "kernel": kernel, "achieved": dk["achieved_tflops"],
        "peak": fp32_peak_of(peaks) / 1e12, "unit": "TFLOP/s", "frac": dk["frac"],
        "traffic": ncu_traffic(kernel),
        "frac_fp32": dk["frac_fp32"], "frac_mufu": dk["frac_mufu"], "frac_evaluated": dk["frac_evaluated"],
        "peak_source": "measured live by darbs_cuda_microbench: the highest of register-operand FFMA, "
                       "immediate-operand FFMA (x2 flops) and packed FFMA2 (x4 flops); MUFU ex2.approx; "
                       "MEASURED_PEAKS.json has no FP32/MUFU entry",
        "peak_ffma_tflops": 2.0 * peaks["ffma_per_s"] / 1e12,
        "peak_mufu_gops": peaks["mufu_per_s"] / 1e9, "peak_sm_mhz": peaks["sm_mhz"],
        "peak_ffma_imm_tflops": 2.0 * peaks["ffma_imm_per_s"] / 1e12,
        "peak_ffma2_tflops": 4.0 * peaks["ffma2_per_s"] / 1e12,
        "algorithmic_work": "flops = V*(13+F_k[+F'_k]) + {9|57}*C per launch with V = sum processed, C = sum "
                            "contributors of that launch (SURVEY 8d); frac = max(flops/peak_fp32, mufu/peak_mufu)/t; "
                            "block-level culling skips visits this count includes, so frac can exceed 1 "
                            "(raised-cosine); frac_evaluated counts only the lane-visits the kernel evaluates "
                            "(32 x composited entries) and is the hardware-utilisation figure (DESIGN.md 3)",
    }


def fp32_peak_of(peaks):
    """FLOP/s of the FP32 pipe: the best of the three instruction forms the micro-benchmark times
    (the render kernels issue FFMA2 where they can, so the packed rate is the honest denominator)."""
    return max(2.0 * peaks["ffma_per_s"], 2.0 * peaks["ffma_imm_per_s"], 4.0 * peaks["ffma2_per_s"])


def dropin_boundary(ctx, darbs, syn, kernels, truth, cam, w, h):
    """The reference-shaped boundary itself: darbs_cuda_forward + darbs_cuda_backward with HOST
    arrays (the darbs::forward / darbs::backward wrappers of INTEGRATION.md option A), all copies
    inside the call: 44 B per splat in, image + aux out; grad_image in, 36 B per splat out.  Inputs
    are pinned host arrays; outputs are pageable numpy arrays, as a caller's std::vector would be.
    Host wall clock around the synchronous calls.  Also the reference's own micro-benchmark sizes
    (benchmarks/bench.cpp:58-75: 200 and 1000 splats, 128 x 128, Gaussian) for small-scene latency."""
    import torch

    def pin(a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).pin_memory().numpy()

    out = {"path": "darbs_cuda_forward + darbs_cuda_backward, DARBS_HOST pointers (splat arrays, images, aux and "
                   "gradients cross PCIe inside the calls)", "per_kernel": {}}
    prims = ctx.realize(np.ascontiguousarray(truth))
    gimg = pin(np.ones((h, w, 3), np.float32))  # bench.cpp:70-71: all-ones upstream gradient
    pairs, secs = 0, 0.0
    for name, (k, psi) in kernels.items():
        pr = ctx.project(k, psi, prims, cam)
        vis = np.flatnonzero(pr["valid"])
        arrs = [pin(pr[key][vis]) for key in ("mu2", "conic", "radius", "depth")] + [pin(prims[vis, 10]), pin(prims[vis, 11:14])]
        nv = int(vis.size)
        tf = tb = 0.0
        reps = 3
        for rep in range(reps + 1):  # the first repetition sizes the staging buffers
            t0 = time.perf_counter()
            ctx.forward(k, *arrs, w, h, (0.0, 0.0, 0.0))
            t1 = time.perf_counter()
            ctx.backward(k, gimg, nv)
            t2 = time.perf_counter()
            if rep:
                tf += t1 - t0
                tb += t2 - t1
        out["per_kernel"][name] = {"splats": nv, "ms_forward": 1e3 * tf / reps, "ms_backward": 1e3 * tb / reps,
                                   "h2d_bytes": 44 * nv + 12 * w * h, "d2h_bytes": 24 * w * h + 36 * nv}
        pairs += reps
        secs += tf + tb
    out["value"] = pairs / secs
    out["unit"] = "forward+backward pairs/s at 1M splats 1080p, host arrays in and out (mean over the 4 kernels)"
    small = {}
    k = kernels["gaussian"][0]
    for n_small in (200, 1000):
        sc = syn.scene_a(n_small, 128, 128, 7)
        arrs = [pin(sc[key]) for key in ("mu2", "conic", "radius", "depth", "opacity", "rgb")]
        g = pin(np.ones((128, 128, 3), np.float32))
        tf = tb = 0.0
        reps = 100
        for rep in range(reps + 5):
            t0 = time.perf_counter()
            ctx.forward(k, *arrs, 128, 128, (0.1, 0.2, 0.3))
            t1 = time.perf_counter()
            ctx.backward(k, g, n_small)
            t2 = time.perf_counter()
            if rep >= 5:
                tf += t1 - t0
                tb += t2 - t1
        small[f"{n_small}_splats_128x128_gaussian"] = {"us_forward": 1e6 * tf / reps, "us_backward": 1e6 * tb / reps}
    out["small_scene_latency"] = small
    return out


def run_config3(args):
    """BASELINE.json configs[3]: 3 M primitives, 64 cameras, 1080p, the views sharded over the GPUs
    (view v -> rank v mod N), one NCCL all-reduce of the 14 N float32 gradients per iteration,
    replicated Adam: fit_scene's iteration (fit3d.cpp:104-184) through darbs_cuda_train_step.  One
    step = one such iteration for each of the four kernels; value = view-iterations per second
    (views x 4 x steps / seconds); the total work is fixed as N grows ("strong")."""
    import torch
    import torch.distributed as dist

    import paper_2501_12369_b200 as darbs
    from paper_2501_12369_b200 import synthetic as syn

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # the communicators' own lines (ranks, NVLS / rings) on stderr: evidence that NCCL carries the exchange
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = darbs.Context(local_rank)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.use_torch_stream()
    ctx.set_exact_decisions(bool(args.exact))
    if world > 1:  # the library's own communicator (NCCL, bound at run time); the id travels over torch's
        ids = [darbs.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        ctx.comm_init(ids[0], rank, world)

    n, w, h, V = args.splats, args.width, args.height, args.views
    truth = syn.scene_b(n, 1)
    init = syn.perturb(truth, 2)
    lrs = torch.from_numpy(syn.learning_rates(init).reshape(-1)).to(dev)
    cams = [syn.orbit_camera(v, V, w, h, args.focal) for v in range(V)]
    truth_d = torch.from_numpy(truth).to(dev)
    bg = (0.0, 0.0, 0.0)
    kernels = {name: (darbs.kernel_preset(name), darbs.default_psi(name)) for name in KERNELS}

    def make_state(views, with_hosts=True):
        st = {}
        for name, (k, psi) in kernels.items():
            targets, hosts = [], []
            for v in views:
                t = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
                ctx.evaluate_view(k, psi, truth_d, cams[v], bg, grad_image=torch.zeros_like(t), image_out=t)
                targets.append(t)
                if with_hosts:  # the end-to-end leg's pinned copies (25 MB per view and kernel)
                    hosts.append(t.cpu().pin_memory().numpy())
            st[name] = dict(params=torch.from_numpy(init).to(dev).clone(), m=torch.zeros(14 * n, device=dev),
                            v=torch.zeros(14 * n, device=dev), grads=torch.zeros((n, 14), device=dev),
                            targets=targets, hosts=hosts, views=list(views), t=0)
        torch.cuda.synchronize()
        return st

    local = list(range(rank, V, world))
    state = make_state(local)
    pending, losses = [0], []

    def iteration(st, name, e2e):
        k, psi = kernels[name]
        s = st[name]
        s["t"] += 1
        view_cams = [cams[v] for v in s["views"]]
        if not e2e:
            ctx.train_step(k, psi, s["params"], s["grads"], s["m"], s["v"], lrs, view_cams, s["targets"], LAMBDA,
                           s["t"], V, bg, want_loss=False)
            return
        # end to end: every view's target image comes from pinned host memory (uploaded under the previous
        # view's render kernels), every view's loss is read back one view late
        if not s["views"]:
            s["grads"].zero_()
        for i, cam in enumerate(view_cams):
            ctx.evaluate_view(k, psi, s["params"], cam, bg, target=s["hosts"][i], lam=LAMBDA, param_grads=s["grads"],
                              want_loss=False, accumulate=i > 0)
            if i + 1 < len(view_cams):
                ctx.prefetch_target(s["hosts"][i + 1])
            pending[0] += 1
            if pending[0] > 1:
                losses.append(ctx.pop_loss())
                pending[0] -= 1
        ctx.allreduce_adam_step(s["params"].view(-1), s["grads"].view(-1), s["m"], s["v"], lrs, s["t"])

    def drain():
        while pending[0] > 0:
            losses.append(ctx.pop_loss())
            pending[0] -= 1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(st, steps, e2e, collective=True):
        if collective:
            barrier()
        else:
            torch.cuda.synchronize()
        l0 = ctx.launch_count()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            for name in KERNELS:
                iteration(st, name, e2e)
        if e2e:
            drain()
        b.record()
        if collective:
            barrier()
        else:
            torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        if collective and world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, ctx.launch_count() - l0

    sampler = ClockSampler(local_rank)
    if rank == 0:
        sampler.start()
    for _ in range(max(args.warmup, 3)):
        for name in KERNELS:
            iteration(state, name, False)
    ms, launches = timed(state, args.steps, False)
    value = V * len(KERNELS) * args.steps / (ms * 1e-3)
    for name in KERNELS:
        iteration(state, name, True)
    drain()
    losses.clear()
    ms_e2e, _ = timed(state, args.steps, True)
    clocks = sampler.stop() if rank == 0 else None
    e2e_value = V * len(KERNELS) * args.steps / (ms_e2e * 1e-3)

    # the dominant kernel's roofline on this rank's first view (Gaussian), stage timers on
    peaks = ctx.microbench()
    roofline = None
    if local:
        ctx.set_stage_timing(True)
        k, psi = kernels["gaussian"]
        s = state["gaussian"]
        ctx.evaluate_view(k, psi, s["params"], cams[local[0]], bg, target=s["targets"][0], lam=LAMBDA,
                          param_grads=s["grads"], accumulate=False)
        st = ctx.stage_times()
        _fw, bw = render_rooflines("gaussian", ctx.work_counters(), st, peaks)
        roofline = roofline_record("render_bwd<gaussian>", bw, peaks)
        roofline["stage_ms_one_view"] = st
        ctx.set_stage_timing(False)

    # strong-scaling reference: the same workload, all views, on rank 0 alone (comm-free library path)
    single = None
    if world > 1 and not args.no_single_gpu_ref:
        barrier()
        if rank == 0:
            ctx.comm_destroy()
            del state
            torch.cuda.empty_cache()
            full = make_state(range(V), with_hosts=False)
            for name in KERNELS:
                iteration(full, name, False)
            steps1 = min(args.steps, 2)
            ms1, _ = timed(full, steps1, False, collective=False)
            single = {"value": V * len(KERNELS) * steps1 / (ms1 * 1e-3), "steps": steps1,
                      "note": "rank 0 alone over all views of the same workload, measured after the timed region"}
        barrier()

    if rank == 0:
        cfg = {
            "workload": f"configs[3]: {n} synthetic 3-D primitives (scene B, SURVEY 8d), {V} orbit cameras {w}x{h}, "
                        f"{(V + world - 1) // world} views per GPU (view v -> rank v mod {world}), full training iteration "
                        f"(preprocess, bin+sort, cull, render fwd, L1 + D-SSIM loss with lambda {LAMBDA}, render bwd, "
                        f"preprocess bwd per view; one all-reduce of the 14 N float32 gradients; Adam) for each of "
                        f"{', '.join(KERNELS)}",
            "splats": n, "width": w, "height": h, "views": V, "views_per_gpu": (V + world - 1) // world,
            "parallelism": f"view-parallel x{world}: darbs_cuda_train_step, ncclAllReduce(sum) of {4 * 14 * n} bytes per "
                           f"iteration in 4 pieces on a side stream, Adam piece by piece" if world > 1 else "single GPU",
            "l2_policy": "inputs larger than L2: every view streams ~1.5 GB of parameters, records, entries and images",
        }
        line = {
            "metric": "train_view_iters_per_sec_3M_splats_1080p_64_views", "value": value,
            "unit": "view-iters/s (fwd+bwd per view, all-reduce + Adam per iteration, mean over the 4 DARBF kernels)",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": cfg, "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": "view-iters/s", "h2d_bytes_per_step": len(KERNELS) * len(local) * 12 * w * h,
                    "d2h_bytes_per_step": len(KERNELS) * len(local) * 32,
                    "path": "per view darbs_cuda_evaluate_view with the target image in pinned host memory "
                            "(darbs_cuda_prefetch_target) and its loss read back (darbs_cuda_pop_loss), then "
                            "darbs_cuda_allreduce_adam_step; per-rank bytes", "losses_read": len(losses)},
            "gpu_launches": int(launches), "roofline": roofline, "single_gpu_same_config": single,
            "exact_decisions": bool(args.exact),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


def cpu_baseline(args, single_thread=True):
    """The reference's CPU code on this box's host cores, bounded to ~10-30 s: one or two training
    iterations per kernel on a 1/16 sample at equal splat density, scaled by 1/16 (the full-size
    figure is `bench.py --impl reference`)."""
    threads = os.cpu_count() or 1
    cpu, orc, kind, truth, cam, init, lrs = cpu_setup(args, fraction=SAMPLE_FRACTION)
    lrs64 = lrs.astype(np.float64)
    total, iters = 0.0, 0
    t_budget = time.perf_counter()
    for name in KERNELS:
        target = cpu_target(orc, cpu, name, truth, cam, threads)
        raw = init.astype(np.float64).copy()
        state = {"m": np.zeros(raw.size), "v": np.zeros(raw.size), "t": 0}
        reps = 2 if time.perf_counter() - t_budget < 20 else 1
        for _ in range(reps):
            dt, _v = cpu_iteration(orc, cpu, name, raw, cam, target, lrs64, state, threads)
            total += dt
            iters += 1
    value = iters / total / SAMPLE_FRACTION
    out = {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
           "sample": f"1/{SAMPLE_FRACTION} of the workload at equal splat density ({truth.shape[0]} primitives, "
                     f"{int(cam[4])}x{int(cam[5])}), {iters} full training iterations over the 4 kernels, "
                     f"value scaled by 1/{SAMPLE_FRACTION}"}
    if single_thread:
        # the same sample on ONE host thread (SURVEY 8d asks for both): one iteration of the cheapest kernel
        name = "half-cosine-sq"
        target = cpu_target(orc, cpu, name, truth, cam, threads)
        raw = init.astype(np.float64).copy()
        state = {"m": np.zeros(raw.size), "v": np.zeros(raw.size), "t": 0}
        dt1, _v = cpu_iteration(orc, cpu, name, raw, cam, target, lrs64, state, 1)
        raw = init.astype(np.float64).copy()
        state = {"m": np.zeros(raw.size), "v": np.zeros(raw.size), "t": 0}
        dtn, _v = cpu_iteration(orc, cpu, name, raw, cam, target, lrs64, state, threads)
        out["single_thread"] = {"kernel": name, "iters_per_s_full_equiv": 1.0 / dt1 / SAMPLE_FRACTION,
                                "all_threads_iters_per_s_full_equiv": 1.0 / dtn / SAMPLE_FRACTION}
    return out


def main():
    args = parse_args()
    if args.impl == "reference" and args.table:
        args.splats = args.splats or 1_000_000
        reference_table(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    elif args.config == 3:
        run_config3(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
