"""The five BASELINE.json workloads as seeded synthetic graph recipes.

The reference measures on SNAP graphs and RMAT 6-17 (PAPER.md tables); those
datasets are not available here, so these seeded generators stand in for them
with the shapes BASELINE.json names:

* ``er4096``   — G(n=4096, p=16/4095), the reference fixture recipe
                 (tests/conftest.py:41-47 er_graph), seed 1.
* ``rmat16``   — generate_rmat(scale=16, ef=16, a/b/c/d=.57/.19/.19/.05,
                 seed=1) (rmat.py:45-72), ids permuted by
                 ``default_rng(2).permutation(n)`` on both endpoints.
* ``lattice2048`` — 2048x2048 grid, 4-neighbour + down-right diagonal,
                 row-major ids; T = 2*2047^2 in closed form.
* ``rmat22`` / ``rmat24`` — as rmat16 at scale 22 / 24.
* ``rmat25`` / ``rmat26`` — capacity cases beyond BASELINE.json (scale 26:
                 2m ≈ 2.1e9 adjacency entries, the int32-id / 32-bit list
                 offset ceiling); checked against the GPU forward count.

RMAT and ER pairs are produced on the device (the PCG64 stream numpy's
default_rng uses, reproduced bit-exactly: tcb_rmat_generate,
tcb_er_generate), as are the lattice's (tcb_lattice_generate); only the RMAT
id permutation (numpy's sequential Fisher-Yates shuffle) comes from the host.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

RMAT_SEED = 1
PERM_SEED = 2
ER_SEED = 1


@dataclass(frozen=True)
class Config:
    name: str
    kind: str          # "er" | "rmat" | "lattice"
    n: int
    scale: int = 0     # rmat
    edge_factor: int = 16
    p: float = 0.0     # er
    side: int = 0      # lattice
    seed: int = 0
    perm_seed: int = 0

    @property
    def raw_pairs(self) -> int:
        if self.kind == "rmat":
            return self.edge_factor * self.n
        if self.kind == "lattice":
            s = self.side
            return 2 * s * (s - 1) + (s - 1) ** 2
        return -1  # er: data dependent


CONFIGS = {
    "er4096": Config("er4096", "er", 4096, p=16 / 4095, seed=ER_SEED),
    "rmat16": Config("rmat16", "rmat", 1 << 16, scale=16, seed=RMAT_SEED,
                     perm_seed=PERM_SEED),
    "lattice2048": Config("lattice2048", "lattice", 2048 * 2048, side=2048),
    "rmat22": Config("rmat22", "rmat", 1 << 22, scale=22, seed=RMAT_SEED,
                     perm_seed=PERM_SEED),
    "rmat24": Config("rmat24", "rmat", 1 << 24, scale=24, seed=RMAT_SEED,
                     perm_seed=PERM_SEED),
    "rmat25": Config("rmat25", "rmat", 1 << 25, scale=25, seed=RMAT_SEED,
                     perm_seed=PERM_SEED),
    "rmat26": Config("rmat26", "rmat", 1 << 26, scale=26, seed=RMAT_SEED,
                     perm_seed=PERM_SEED),
}


def er_pairs(n: int, p: float, seed: int) -> np.ndarray:
    """Reference fixture recipe (tests/conftest.py:41-47): u<v pairs with
    default_rng(seed).random((n, n)) < p over the strict upper triangle."""
    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < p
    iu = np.triu_indices(n, k=1)
    sel = mask[iu]
    return np.stack([iu[0][sel], iu[1][sel]], axis=1).astype(np.int64)


def er_pairs_device(n: int, p: float, seed: int, device=None):
    """er_pairs on the GPU (tcb_er_generate): torch int64 [k, 2]."""
    import ctypes

    import torch

    from . import _lib
    from .rmat import _hi_lo, pcg64_seed_state
    ctx = _lib.context(device)
    dev = torch.device("cuda", ctx.device)
    cap = max(1, n * (n - 1) // 2)
    pairs = torch.empty((cap, 2), dtype=torch.int64, device=dev)
    st, inc = pcg64_seed_state(seed)
    k = ctypes.c_int64(0)
    ctx.check(ctx.lib.tcb_er_generate(ctx.h, n, float(p), *_hi_lo(st), *_hi_lo(inc),
                                      _lib.ptr(pairs), ctypes.byref(k)))
    return pairs[: int(k.value)]


def lattice_pairs_device(side: int, device=None):
    """lattice_pairs on the GPU (tcb_lattice_generate): torch int64 [k, 2]."""
    import torch

    from . import _lib
    ctx = _lib.context(device)
    dev = torch.device("cuda", ctx.device)
    k = 2 * side * (side - 1) + (side - 1) ** 2
    pairs = torch.empty((max(k, 1), 2), dtype=torch.int64, device=dev)
    ctx.check(ctx.lib.tcb_lattice_generate(ctx.h, side, _lib.ptr(pairs)))
    return pairs[:k]


def id_permutation(n: int, seed: int) -> np.ndarray:
    """The seeded vertex relabeling applied to RMAT endpoints: new = perm[old]."""
    return np.random.default_rng(seed).permutation(n).astype(np.int64)


def lattice_pairs(side: int) -> np.ndarray:
    """(r,c)-(r,c+1), (r,c)-(r+1,c), (r,c)-(r+1,c+1), ids r*side+c."""
    r, c = np.meshgrid(np.arange(side, dtype=np.int64),
                       np.arange(side, dtype=np.int64), indexing="ij")
    vid = r * side + c
    right = np.stack([vid[:, :-1].ravel(), vid[:, 1:].ravel()], axis=1)
    down = np.stack([vid[:-1, :].ravel(), vid[1:, :].ravel()], axis=1)
    diag = np.stack([vid[:-1, :-1].ravel(), vid[1:, 1:].ravel()], axis=1)
    return np.concatenate([right, down, diag], axis=0)


def lattice_closed_form(side: int) -> dict:
    """Closed forms verified against the oracle."""
    s = side
    return dict(m=2 * s * (s - 1) + (s - 1) ** 2, T=2 * (s - 1) ** 2,
                max_level=s - 1, cover=s * (s - 1), components=1)


def build_device_graph(cfg: "Config | str", device=None):
    """Materialise a config as a DeviceGraph: pairs generated in HBM (PCG64
    replay for RMAT / ER, closed form for the lattice; RMAT ids permuted by
    the host permutation), then the device CSR build (tcb_csr_build)."""
    import torch

    from .graph import normalize_device
    from .rmat import RmatParams, rmat_pairs_device

    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if cfg.kind == "rmat":
        perm = id_permutation(cfg.n, cfg.perm_seed)
        pairs = rmat_pairs_device(RmatParams(scale=cfg.scale, edge_factor=cfg.edge_factor,
                                             seed=cfg.seed), perm=perm, device=dev.index)
    elif cfg.kind == "er":
        pairs = er_pairs_device(cfg.n, cfg.p, cfg.seed, device=dev.index)
    else:
        pairs = lattice_pairs_device(cfg.side, device=dev.index)
    with torch.cuda.device(dev):
        dg = normalize_device(cfg.n, pairs)
    del pairs
    return dg
