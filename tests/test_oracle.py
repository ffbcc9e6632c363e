"""The CPU oracle (oracle/) against the reference's own outputs.

Pins the C restatement before it is trusted as the checker: every hot-path
output of every golden case (produced by importing the reference, see
tests/golden/make_golden.py) must match bit for bit.
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle
from conftest import SMALL_CASES, SMALL_IDS, config_goldens
from paper_2403_02997_b200 import configs as C


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", SMALL_CASES, ids=SMALL_IDS)
def test_oracle_matches_reference_small(case):
    row, nb, eu, ev = oracle.normalize(case.n, case.pairs)
    assert np.array_equal(row, case.row)
    assert np.array_equal(nb, case.nb)
    assert np.array_equal(eu, case.eu) and np.array_equal(ev, case.ev)
    out = oracle.run(case.n, row, nb, eu, ev, threads=2)
    assert np.array_equal(out["level"], case.level)
    assert np.array_equal(out["parent"], case.parent)
    assert np.array_equal(out["edge_class"], case.edge_class)
    assert out["components"] == case.components
    assert out["max_level"] == case.max_level
    assert np.array_equal(out["cover"], case.cover)
    assert (out["T"], out["c1"], out["c2"]) == (case.T, case.c1, case.c2)
    assert oracle.cetc_count(row, nb, out["level"], case.n) == case.T
    drow, dnb = oracle.degree_order(case.n, row, eu, ev)
    assert np.array_equal(drow, case.deg_row) and np.array_equal(dnb, case.deg_nb)
    if case.n <= 80:
        assert oracle.brute_count(case.n, row, nb) == case.T


def test_pcg64_stream_matches_numpy():
    for seed in (0, 1, 2, 123):
        ref = np.random.default_rng(seed).random(1000)
        assert np.array_equal(oracle.pcg64_doubles(seed, 1000), ref)
    # jump-ahead
    ref = np.random.default_rng(7).random(5000)[4321:]
    assert np.array_equal(oracle.pcg64_doubles(7, len(ref), skip=4321), ref)


@pytest.mark.parametrize("name,scale,ef,seed", [
    ("rmat4", 4, 8, 4), ("rmat5", 5, 8, 5), ("rmat6", 6, 8, 6),
    ("rmat7_9", 7, 16, 9), ("rmat8_77", 8, 16, 77), ("rmat10_42", 10, 16, 42)])
def test_oracle_rmat_matches_reference_pairs(name, scale, ef, seed):
    case = next(c for c in SMALL_CASES if c.name == name)
    assert np.array_equal(oracle.rmat_pairs(scale, ef, seed=seed), case.pairs)


def test_config_er4096():
    g = config_goldens()["er4096"]
    cfg = C.CONFIGS["er4096"]
    row, nb, eu, ev = oracle.normalize(cfg.n, C.er_pairs(cfg.n, cfg.p, cfg.seed))
    assert sha(row) == g["row_offsets_sha"] and sha(nb) == g["neighbors_sha"]
    out = oracle.run(cfg.n, row, nb, eu, ev, threads=4)
    assert out["level"].tolist() == g["level_int8"]
    assert sha(out["level"].astype(np.int32)) == g["level_sha"]
    assert sha(out["cover"].astype(np.int32)) == g["cover_sha"]
    assert (out["T"], out["c1"], out["c2"]) == (g["T"], g["c1"], g["c2"])


@pytest.mark.slow
def test_config_rmat16():
    g = config_goldens()["rmat16"]
    cfg = C.CONFIGS["rmat16"]
    perm = C.id_permutation(cfg.n, cfg.perm_seed)
    pairs = oracle.rmat_pairs(cfg.scale, cfg.edge_factor, seed=cfg.seed, perm=perm)
    row, nb, eu, ev = oracle.normalize(cfg.n, pairs)
    assert sha(row) == g["row_offsets_sha"] and sha(nb) == g["neighbors_sha"]
    out = oracle.run(cfg.n, row, nb, eu, ev, threads=oracle.max_threads())
    assert sha(out["level"].astype(np.int32)) == g["level_sha"]
    assert sha(out["cover"].astype(np.int32)) == g["cover_sha"]
    assert (out["T"], out["c1"], out["c2"]) == (g["T"], g["c1"], g["c2"])
    assert (out["components"], out["max_level"]) == (g["components"], g["max_level"])


def test_lattice_closed_form_small():
    for side in (2, 3, 5, 17, 64):
        pairs = C.lattice_pairs(side)
        n = side * side
        row, nb, eu, ev = oracle.normalize(n, pairs)
        out = oracle.run(n, row, nb, eu, ev)
        cf = C.lattice_closed_form(side)
        assert len(eu) == cf["m"]
        assert out["T"] == cf["T"]
        assert out["max_level"] == cf["max_level"]
        assert len(out["cover"]) == cf["cover"]
        r, c = np.divmod(np.arange(n), side)
        assert np.array_equal(out["level"], np.maximum(r, c))
