"""Host-side logic that needs no GPU: argument validation and ingest,
mirroring the reference's own tests (test_graph.py, test_rmat.py,
test_parallel.py)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2403_02997_b200 as tb
from paper_2403_02997_b200 import configs as C


class TestParse:
    def test_triangle_literal(self):
        el = tb.parse_edge_list("0 1\n1 2\n0 2\n")
        assert el.n == 3
        assert el.edges.tolist() == [[0, 1], [1, 2], [0, 2]]

    def test_sparse_ids_relabeled(self):
        el = tb.parse_edge_list("# c\n5 7\n")
        assert el.n == 2 and el.edges.tolist() == [[0, 1]]
        assert el.original_ids.tolist() == [5, 7]

    def test_first_appearance_order(self):
        el = tb.parse_edge_list("9 4\n4 2\n")
        assert el.original_ids.tolist() == [9, 4, 2]
        assert el.edges.tolist() == [[0, 1], [1, 2]]

    def test_comments_blank_bytes_empty(self):
        assert tb.parse_edge_list("% h\n\n  \n0 1\n# t\n").n == 2
        assert tb.parse_edge_list(b"0 1\n").n == 2
        el = tb.parse_edge_list("")
        assert el.n == 0 and len(el.edges) == 0

    @pytest.mark.parametrize("text,frag", [("0 1 2\n", "line 1"), ("0\n", "line 1"),
                                           ("0 x\n", "non-integer"), ("0 1\n-1 2\n", "line 2")])
    def test_malformed(self, text, frag):
        with pytest.raises(tb.ParseError, match=frag):
            tb.parse_edge_list(text)

    def test_edge_list_range_check(self):
        with pytest.raises(ValueError):
            tb.EdgeList(n=2, edges=np.array([[0, 5]]))


class TestParams:
    @pytest.mark.parametrize("kw", [dict(scale=0), dict(scale=63), dict(scale=5, edge_factor=0),
                                    dict(scale=5, a=0.5, b=0.5, c=0.5, d=0.5),
                                    dict(scale=5, a=-0.1, b=0.5, c=0.3, d=0.3)])
    def test_rmat_invalid(self, kw):
        with pytest.raises(ValueError):
            tb.RmatParams(**kw)

    def test_parallel_config(self):
        with pytest.raises(ValueError):
            tb.ParallelConfig(workers=0)
        with pytest.raises(ValueError):
            tb.ParallelConfig(workers=2, chunk=0)
        assert tb.ParallelConfig(workers=2).ranges(0) == []
        r = tb.ParallelConfig(workers=2).ranges(17)
        assert r[0] == (0, 3) and r[-1][1] == 17
        assert tb.ParallelConfig(workers=1, chunk=5).ranges(12) == [(0, 5), (5, 10), (10, 12)]

    def test_unknown_ids(self):
        with pytest.raises(ValueError, match="unknown"):
            tb.count_sequential("NOPE", None)
        with pytest.raises(ValueError, match="unknown"):
            tb.tc_par("NOPE", None, tb.ParallelConfig())

    def test_registry_names(self):
        # the reference's cetc-family group (bench.py:42-43): every id that
        # starts with "CETC" in SEQUENTIAL_IDS (sequential.py:261-267) and
        # PARALLEL_IDS (parallel.py:151)
        assert sorted(tb.SEQUENTIAL_IDS) == sorted([
            "CETC-Seq", "CETC-Seq-D", "CETC-Seq-FE", "CETC-Seq-S", "CETC-Seq-SD", "CETC-Seq-SR"])
        assert list(tb.PARALLEL_IDS) == ["CETC-SM"]
        assert tb.COVER_RATIO_THRESHOLD == 0.7


class TestConfigs:
    def test_shapes(self):
        assert C.CONFIGS["rmat24"].n == 1 << 24
        assert C.CONFIGS["rmat16"].raw_pairs == 1 << 20
        assert C.CONFIGS["lattice2048"].raw_pairs == 12_574_721
        cf = C.lattice_closed_form(2048)
        assert cf["T"] == 8_380_418 and cf["m"] == 12_574_721

    def test_lattice_pairs(self):
        p = C.lattice_pairs(3)
        assert len(p) == 2 * 3 * 2 + 4
        assert (p[:, 0] < p[:, 1]).all()

    def test_er_recipe_matches_fixture_rule(self):
        p = C.er_pairs(30, 0.25, 0)
        assert (p[:, 0] < p[:, 1]).all()
        rng = np.random.default_rng(0)
        mask = rng.random((30, 30)) < 0.25
        iu = np.triu_indices(30, k=1)
        assert len(p) == int(mask[iu].sum())

    def test_permutation_is_seeded(self):
        a = C.id_permutation(1000, 2)
        assert np.array_equal(a, C.id_permutation(1000, 2))
        assert sorted(a.tolist()) == list(range(1000))
