"""The view-parallel trainer on a GPU without any manual stream set-up (torch's ops and
the library's kernels must share one stream; bind_context binds the context itself).  One rank:
the all-reduce is the identity, the rest of the iteration is what every rank of an N-GPU job runs.
The CPU oracle supplies the serial answer (fit3d.cpp:104-184)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_trainer_matches_the_serial_view_loop(port, darbs):
    import torch

    from oracle.cpu import Scene
    from paper_2501_12369_b200 import synthetic as syn
    from paper_2501_12369_b200.multiview import ViewParallelTrainer, bind_context

    name, n, n_views, w, h = "half-cosine-sq", 400, 3, 64, 48
    k, gk, psi = port.preset(name), darbs.kernel_preset(name), port.default_psi(name)
    truth = syn.scene_b(n, 1, half_extent=(0.5, 0.4, 0.4), scale_range=(0.02, 0.06))
    init = syn.perturb(truth, 2)
    cams = [syn.orbit_camera(v, n_views, w, h, 60.0) for v in range(n_views)]
    lrs = syn.learning_rates(init)

    def scene_of(raw, cam):
        prims = port.realize(raw.astype(np.float64))
        st, pr = port.project(k, psi, prims, cam)
        vis = np.flatnonzero(pr["valid"]).astype(np.int32)
        return prims, vis, Scene(pr["mu2"][vis], None, pr["conic"][vis], pr["radius"][vis], pr["depth"][vis],
                                 prims[vis, 10], prims[vis, 11:14])

    targets = [port.forward(k, scene_of(truth, cam)[2], w, h, (0, 0, 0))["image"].astype(np.float32) for cam in cams]
    # serial reference iteration: gradients summed over views, one Adam step
    g_ref = np.zeros((n, 14))
    for cam, tgt in zip(cams, targets):
        prims, vis, s = scene_of(init, cam)
        fr = port.forward(k, s, w, h, (0, 0, 0), keep=True)
        st, _vals, gimg = port.loss_total(fr["image"], tgt.astype(np.float64), 0.2)
        st, sg = port.backward(fr["handle"], k, gimg, s)
        port.forward_free(fr["handle"])
        g_ref += port.param_grads(psi, vis, sg, s.conic, s.opacity, s.rgb, prims, cam)
    st, p_ref, _m, _v = port.adam_step(init.astype(np.float64).reshape(-1), g_ref.reshape(-1), np.zeros(14 * n),
                                       np.zeros(14 * n), lrs.astype(np.float64).reshape(-1), 1)

    dev = torch.device("cuda", 0)
    side = torch.cuda.Stream(dev)  # NOT the stream the context was created on, and no use_torch_stream() here
    with darbs.Context(0) as ctx, torch.cuda.stream(side):
        evaluate, adam = bind_context(ctx, gk, psi, cams, [torch.from_numpy(t).to(dev) for t in targets],
                                      want_loss=False)
        tr = ViewParallelTrainer(torch.from_numpy(init).to(dev), torch.from_numpy(lrs).to(dev), n_views, evaluate, adam)
        tr.step(want_loss=False)
        grads = tr.grads.cpu().numpy()
        params = tr.params.cpu().numpy()
    floor = 2e-4 * max(1.0, np.abs(g_ref).max())
    err = np.abs(grads - g_ref) / np.maximum(np.maximum(np.abs(grads), np.abs(g_ref)), floor)
    assert err.max() <= 2e-3, err.max()
    # the first Adam step moves every parameter by lr * sign(g) (optim.hpp:24-39): compare where the
    # gradient is well away from zero
    big = np.abs(g_ref).reshape(-1) > 1e-6
    assert np.abs(params.reshape(-1) - p_ref)[big].max() <= 1e-5


def test_train_step_matches_the_view_loop_with_a_one_rank_communicator(darbs):
    """darbs_cuda_train_step (the C ABI's fit_scene iteration: local views, NCCL all-reduce in pieces
    on a side stream, Adam piece by piece) against the same iteration spelled out with
    evaluate_view + adam_step.  A world-size-1 NCCL communicator makes the all-reduce the identity,
    so the NCCL call site, its stream hand-off and the piecewise Adam all run on one GPU; in the
    deterministic mode the two spellings must agree bit for bit."""
    import torch

    from paper_2501_12369_b200 import synthetic as syn

    name, n, n_views, w, h = "gaussian", 3000, 3, 96, 64
    gk, psi = darbs.kernel_preset(name), darbs.default_psi(name)
    truth = syn.scene_b(n, 1, half_extent=(0.5, 0.4, 0.4), scale_range=(0.01, 0.04))
    init = syn.perturb(truth, 2)
    cams = [syn.orbit_camera(v, n_views, w, h, 90.0) for v in range(n_views)]
    dev = torch.device("cuda", 0)
    lrs = torch.from_numpy(syn.learning_rates(init).reshape(-1)).to(dev)
    results = []
    for use_train_step in (False, True):
        with darbs.Context(0) as ctx:
            ctx.use_torch_stream()
            ctx.set_deterministic(True)
            truth_d = torch.from_numpy(truth).to(dev)
            targets = []
            for cam in cams:
                t = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
                ctx.evaluate_view(gk, psi, truth_d, cam, (0, 0, 0), grad_image=torch.zeros_like(t), image_out=t)
                targets.append(t)
            p = torch.from_numpy(init).to(dev).clone()
            g = torch.zeros_like(p)
            m, v = torch.zeros(14 * n, device=dev), torch.zeros(14 * n, device=dev)
            losses = []
            if use_train_step:
                ctx.comm_init(darbs.comm_unique_id(), 0, 1)
            for it in (1, 2, 3):
                if use_train_step:
                    losses.append(ctx.train_step(gk, psi, p, g, m, v, lrs, cams, targets, 0.2, it, n_views))
                else:
                    sums = np.zeros(4)
                    for i, cam in enumerate(cams):
                        sums += ctx.evaluate_view(gk, psi, p, cam, (0, 0, 0), target=targets[i], lam=0.2, param_grads=g,
                                                  accumulate=i > 0)
                    ctx.adam_step(p.view(-1), g.view(-1), m, v, lrs, it)
                    losses.append(tuple(sums / n_views))
            torch.cuda.synchronize()
            results.append((p.cpu().numpy(), g.cpu().numpy(), np.array(losses)))
    (p0, g0, l0), (p1, g1, l1) = results
    assert np.array_equal(g0, g1)
    assert np.array_equal(p0, p1)
    assert np.abs(l0 - l1).max() <= 1e-12 * np.abs(l0).max()
    assert np.abs(p0 - init).max() > 1e-5 and l0[2, 0] < l0[0, 0]  # it did train
