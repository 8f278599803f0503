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
