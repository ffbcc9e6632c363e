"""RMAT input synthesis on the device (drop-in for tricount.rmat).

``generate_rmat`` returns the reference's pairs bit-for-bit (rmat.py:45-72):
the kernel replays the PCG64 stream that numpy.random.default_rng(seed)
draws from, jumping each thread to its own draw index, instead of looping
over 1 Mi-pair blocks on the host.  ``rmat_pairs_device`` keeps the pairs in
HBM (optionally id-permuted) for the device CSR build.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import EdgeList

__all__ = ["RmatParams", "generate_rmat", "rmat_pairs_device", "pcg64_seed_state"]


@dataclass(frozen=True)
class RmatParams:
    """Quadrant probabilities and size (rmat.py:15-42, same validation)."""

    scale: int
    edge_factor: int = 16
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    d: float = 0.05
    seed: int = 1

    def __post_init__(self):
        if self.scale < 1:
            raise ValueError("scale must be >= 1")
        if self.scale > 62:
            raise ValueError("scale too large for 64-bit vertex ids")
        if self.edge_factor < 1:
            raise ValueError("edge_factor must be >= 1")
        probs = (self.a, self.b, self.c, self.d)
        if any(p < 0 for p in probs):
            raise ValueError("quadrant probabilities must be non-negative")
        if abs(sum(probs) - 1.0) > 1e-9:
            raise ValueError("quadrant probabilities must sum to 1")


def pcg64_seed_state(seed: int) -> tuple[int, int]:
    """(state, inc) that numpy.random.default_rng(seed)'s PCG64 starts from."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


def _hi_lo(x: int):
    return (x >> 64) & 0xFFFFFFFFFFFFFFFF, x & 0xFFFFFFFFFFFFFFFF


def rmat_pairs_device(params: RmatParams, perm=None, device=None):
    """edge_factor * 2^scale pairs as a torch int64 [k, 2] CUDA tensor.
    ``perm`` (length 2^scale) relabels both endpoints: new = perm[old]."""
    import torch
    if params.scale > 30:
        raise ValueError("device generator supports scale <= 30 (int32 ids)")
    ctx = _lib.context(device)
    dev = torch.device("cuda", ctx.device)
    n = 1 << params.scale
    total = params.edge_factor * n
    pairs = torch.empty((total, 2), dtype=torch.int64, device=dev)
    p = None
    if perm is not None:
        p = torch.as_tensor(np.ascontiguousarray(perm, dtype=np.int64)).to(dev) \
            if not isinstance(perm, torch.Tensor) else perm.to(dev, torch.int64).contiguous()
        if p.numel() != n:
            raise ValueError("perm must have 2^scale entries")
    s, inc = pcg64_seed_state(params.seed)
    ctx.check(ctx.lib.tcb_rmat_generate(ctx.h, params.scale, params.edge_factor,
                                        params.a, params.b, params.c, *_hi_lo(s),
                                        *_hi_lo(inc), _lib.ptr(p), _lib.ptr(pairs)))
    return pairs


def generate_rmat(params: RmatParams) -> EdgeList:
    """Sample edge_factor * 2^scale directed pairs by recursive quadrant
    choice, MSB first; bit-identical to the reference for the same seed."""
    pairs = rmat_pairs_device(params)
    return EdgeList(n=1 << params.scale, edges=pairs.cpu().numpy())
