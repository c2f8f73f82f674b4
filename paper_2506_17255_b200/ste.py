"""Fake-compress straight-through estimator (§3.3, Figure 4b).

"Each original weight (a trainable parameter) is first compressed using the AbsMaxMin sketch,
updating the sketch states.  Then, weights are retrieved from sketch states waiting for
computation, which forms a fake-compress procedure.  This procedure does not track the gradient,
and the gradient from the preceding computation part estimates each weight gradient"
(PAPER.md:299-302).  Forward = usk_build + usk_reconstruct of the CURRENT weights (every call,
so bindings may migrate as the weights change); backward = identity.  Both run in libusk's CUDA
kernels; this module is autograd plumbing only.  Finetuning itself is out of scope.

The aggregated-gradient baseline (Figure 4a) is usk.aggregate_grad.
"""
from __future__ import annotations

import torch

from . import usk


class FakeCompress(torch.autograd.Function):
    """W -> W' = reconstruct(build(W)); dL/dW := dL/dW' (straight-through)."""

    @staticmethod
    def forward(ctx, W, plan, layer, sketch):
        usk.build(plan, [W.detach().contiguous()], sketch, layer_ids=[layer])
        Wp = torch.empty(W.shape, dtype=W.dtype, device=W.device)  # dense row-major, whatever W's strides
        usk.reconstruct(plan, sketch, layer, Wp)
        return Wp

    @staticmethod
    def backward(ctx, grad_out):
        return grad_out, None, None, None


def fake_compress(W: torch.Tensor, plan, layer: int, sketch: torch.Tensor) -> torch.Tensor:
    """Fake-compressed copy of the weight W ([out, in], plan dtype, CUDA) of `layer` with a
    straight-through gradient; `sketch` receives the layer's states (plan.new_sketch())."""
    return FakeCompress.apply(W, plan, layer, sketch)
