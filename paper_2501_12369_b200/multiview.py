"""View-parallel training iteration: fit_scene's loop (src/fit3d.cpp:104-184) sharded by camera.

The reference walks the views serially and meets only at ``grads[owner] += ...``
(fit3d.cpp:148-158); the reported loss is the view mean (fit3d.cpp:161-165).  Here view ``v``
belongs to rank ``v mod world``, every rank keeps a full replica of the 14·N raw
parameters and Adam state, accumulates its local views into one 14·N float32 gradient buffer, and
one all-reduce (SUM, no 1/V scaling) over ``torch.distributed`` — NCCL over NVLink on the GPUs,
gloo in the CPU tests — makes the gradients identical everywhere before the replicated Adam step.
There is no other exchange on the path.

The per-view evaluation and the Adam update are callables so that the host logic can be tested
on CPU with world_size 2 (tests/test_multiview_gloo.py); :func:`bind_context` supplies the
product ones, which call the C ABI (darbs_cuda_evaluate_view / darbs_cuda_adam_step).
"""
from __future__ import annotations

from typing import Callable, Sequence


def local_views(n_views: int, world: int, rank: int) -> list[int]:
    """Static round-robin assignment view v -> rank v mod world."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return list(range(rank, n_views, world))


class ViewParallelTrainer:
    """One replica of the scene parameters; ``step`` is one fit_scene iteration over all views.

    evaluate(view, params, grads) -> (total, l1, dssim, mse): adds the view's parameter gradients
        into ``grads`` in place (darbs_cuda_evaluate_view's contract).
    adam(params, grads, m, v, lrs, t): in-place update (darbs_cuda_adam_step's contract).
    """

    def __init__(self, params, lrs, n_views: int, evaluate: Callable, adam: Callable, *, world: int = 1,
                 rank: int = 0, group=None):
        import torch

        self.torch = torch
        self.params, self.lrs = params, lrs
        self.grads = torch.zeros_like(params)
        self.m = torch.zeros_like(params)
        self.v = torch.zeros_like(params)
        self.n_views, self.world, self.rank, self.group = n_views, world, rank, group
        self.views = local_views(n_views, world, rank)
        self.evaluate, self.adam = evaluate, adam
        self.t = 0

    def reduce_gradients(self):
        """The all-reduce site: fit3d.cpp:148-158's ``+=`` over views, across ranks."""
        if self.world > 1:
            import torch.distributed as dist

            dist.all_reduce(self.grads, op=dist.ReduceOp.SUM, group=self.group)

    def reduce_loss(self, sums: Sequence[float]):
        """View-mean of (total, l1, dssim, mse), fit3d.cpp:161-165."""
        t = self.torch.tensor(list(sums), dtype=self.torch.float64, device=self.grads.device)
        if self.world > 1:
            import torch.distributed as dist

            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return tuple(float(x) / self.n_views for x in t.tolist())

    def step(self, want_loss: bool = True):
        self.grads.zero_()
        sums = [0.0, 0.0, 0.0, 0.0]
        for view in self.views:
            loss = self.evaluate(view, self.params, self.grads)
            if want_loss and loss is not None:
                sums = [a + b for a, b in zip(sums, loss)]
        self.reduce_gradients()
        self.t += 1
        self.adam(self.params, self.grads, self.m, self.v, self.lrs, self.t)
        return self.reduce_loss(sums) if want_loss else None


def bind_context(ctx, kernel, psi: float, cameras, targets, background=(0.0, 0.0, 0.0), lam: float = 0.2,
                 want_loss: bool = True):
    """(evaluate, adam) that run on a :class:`paper_2501_12369_b200.Context` through the C ABI.
    ``targets[v]`` may be a CUDA tensor (device-resident) or a pinned host array (DARBS_HOST);
    ``lam`` defaults to FitConfig::lambda (include/darbs/fit_common.hpp:16).

    The trainer mixes torch ops (``grads.zero_()``, the NCCL all-reduce) with the library's
    kernels; both must run on ONE stream or nothing orders the all-reduce behind the last view's
    gradient kernel.  The context is therefore bound to torch's current stream here, and again in
    every call (the caller may have switched streams since)."""
    ctx.use_torch_stream()

    def evaluate(view, params, grads):
        ctx.use_torch_stream()
        tgt = targets[view]
        if hasattr(tgt, "is_cuda") and not tgt.is_cuda:
            tgt = tgt.numpy()
        return ctx.evaluate_view(kernel, psi, params, cameras[view], background, target=tgt, lam=lam,
                                 param_grads=grads, want_loss=want_loss)

    def adam(params, grads, m, v, lrs, t):
        ctx.use_torch_stream()
        ctx.adam_step(params.view(-1), grads.view(-1), m.view(-1), v.view(-1), lrs.view(-1), t)

    return evaluate, adam
