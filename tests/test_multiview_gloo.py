"""World-size-2 test (gloo, CPU) of the view-parallel training iteration's host logic
(paper_2501_12369_b200/multiview.py): view -> rank assignment, SUM all-reduce of the 14N gradient
buffer, view-mean loss, replicated Adam.  The per-view evaluation is supplied by the CPU oracle
here (the checker standing in for the GPU call, which needs a B200); the serial answer is
fit_scene's own loop order, src/fit3d.cpp:104-184.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

N_PRIMS, N_VIEWS, W, H, KERNEL = 150, 5, 48, 40, "half-cosine-sq"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup():
    sys.path.insert(0, ROOT)
    from oracle import cpu
    from paper_2501_12369_b200 import synthetic as syn

    orc = cpu.load("port")
    k = orc.preset(KERNEL)
    psi = orc.default_psi(KERNEL)
    truth = syn.scene_b(N_PRIMS, 1, half_extent=(0.5, 0.4, 0.4), scale_range=(0.02, 0.06))
    init = syn.perturb(truth, 2)
    cams = [syn.orbit_camera(v, N_VIEWS, W, H, 60.0) for v in range(N_VIEWS)]
    lrs = syn.learning_rates(init)

    def render(raw, cam):
        prims = orc.realize(raw.astype(np.float64))
        st, pr = orc.project(k, psi, prims, cam)
        vis = np.flatnonzero(pr["valid"]).astype(np.int32)
        s = cpu.Scene(pr["mu2"][vis], None, pr["conic"][vis], pr["radius"][vis], pr["depth"][vis], prims[vis, 10],
                      prims[vis, 11:14])
        return prims, vis, s

    targets = []
    for cam in cams:
        _, _, s = render(truth, cam)
        targets.append(orc.forward(k, s, W, H, (0, 0, 0))["image"])

    def evaluate_np(view, raw, grads):
        """fit3d.cpp:108-159 for one view with the L1 loss (lambda = 0); grads += in place."""
        prims, vis, s = render(raw, cams[view])
        fr = orc.forward(k, s, W, H, (0, 0, 0), keep=True)
        d = fr["image"] - targets[view]
        st, sg = orc.backward(fr["handle"], k, np.sign(d) / d.size, s)
        orc.forward_free(fr["handle"])
        grads += orc.param_grads(psi, vis, sg, s.conic, s.opacity, s.rgb, prims, cams[view])
        l1 = float(np.abs(d).mean())
        return (l1, l1, 0.0, float((d * d).mean()))

    def adam_np(p, g, m, v, lr, t):
        st, p2, m2, v2 = orc.adam_step(p.reshape(-1), g.reshape(-1), m.reshape(-1), v.reshape(-1), lr.reshape(-1), t)
        p[...] = p2.reshape(p.shape)
        m[...] = m2.reshape(m.shape)
        v[...] = v2.reshape(v.shape)

    return init.astype(np.float64), lrs.astype(np.float64), evaluate_np, adam_np


def _serial(steps):
    init, lrs, evaluate_np, adam_np = _setup()
    p, m, v = init.copy(), np.zeros_like(init), np.zeros_like(init)
    losses = []
    for t in range(1, steps + 1):
        g = np.zeros_like(p)
        sums = np.zeros(4)
        for view in range(N_VIEWS):  # the reference's serial view order
            sums += evaluate_np(view, p, g)
        adam_np(p, g, m, v, lrs, t)
        losses.append(sums / N_VIEWS)
    return p, np.array(losses)


def _worker(rank, world, port, steps, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        init, lrs, evaluate_np, adam_np = _setup()
        from paper_2501_12369_b200.multiview import ViewParallelTrainer, local_views

        def evaluate(view, params, grads):
            assert view in local_views(N_VIEWS, world, rank)
            return evaluate_np(view, params.numpy(), grads.numpy())

        def adam(p, g, m, v, lr, t):
            adam_np(p.numpy(), g.numpy(), m.numpy(), v.numpy(), lr.numpy(), t)

        tr = ViewParallelTrainer(torch.from_numpy(init.copy()), torch.from_numpy(lrs), N_VIEWS, evaluate, adam,
                                 world=world, rank=rank)
        losses = [tr.step() for _ in range(steps)]
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), params=tr.params.numpy(), losses=np.array(losses),
                 views=np.array(tr.views))
    finally:
        dist.destroy_process_group()


def test_local_views_partition():
    from paper_2501_12369_b200.multiview import local_views

    for world in (1, 2, 3, 8):
        seen = sorted(v for r in range(world) for v in local_views(64, world, r))
        assert seen == list(range(64))
        assert all(v % world == r for r in range(world) for v in local_views(64, world, r))
    assert local_views(3, 8, 5) == []
    with pytest.raises(ValueError):
        local_views(4, 2, 2)


def test_two_ranks_match_the_serial_view_loop(tmp_path):
    import torch.multiprocessing as mp

    steps, world = 2, 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, steps, str(tmp_path)), nprocs=world, join=True)
    ref_p, ref_l = _serial(steps)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    assert r0["views"].tolist() == [0, 2, 4] and r1["views"].tolist() == [1, 3]
    # replicas stay bit-identical: same all-reduced gradients, same Adam
    assert np.array_equal(r0["params"], r1["params"])
    assert np.array_equal(r0["losses"], r1["losses"])
    # and equal to the serial loop up to the FP64 summation order over views (SURVEY 8e parity note)
    assert np.abs(r0["params"] - ref_p).max() <= 1e-9
    assert np.abs(r0["losses"] - ref_l).max() <= 1e-12
    assert np.abs(ref_p - _setup()[0]).max() > 1e-5  # the steps did move the parameters


def test_four_ranks_with_uneven_view_counts(tmp_path):
    """World size 4 over 5 views: ranks own 2, 1, 1, 1 views (view v -> rank v mod 4), one rank more
    than the others; the all-reduce is a SUM without any per-rank weight, so the result is still the
    serial loop's (fit3d.cpp:148-158 sums the views; :161-165 divides the loss by the view count)."""
    import torch.multiprocessing as mp

    steps, world = 2, 4
    port = _free_port()
    mp.spawn(_worker, args=(world, port, steps, str(tmp_path)), nprocs=world, join=True)
    ref_p, ref_l = _serial(steps)
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert [r["views"].tolist() for r in ranks] == [[0, 4], [1], [2], [3]]
    for r in ranks[1:]:
        assert np.array_equal(r["params"], ranks[0]["params"])
        assert np.array_equal(r["losses"], ranks[0]["losses"])
    assert np.abs(ranks[0]["params"] - ref_p).max() <= 1e-9
    assert np.abs(ranks[0]["losses"] - ref_l).max() <= 1e-12


def test_more_ranks_than_views_leaves_idle_ranks_consistent(tmp_path):
    """A rank without a view contributes zeros to the sum and still ends with the same parameters."""
    from paper_2501_12369_b200.multiview import local_views

    assert local_views(N_VIEWS, 8, 6) == [] and local_views(N_VIEWS, 8, 4) == [4]
