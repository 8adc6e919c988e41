"""The engine's native generators are bit-identical to the reference's
(bench/generators.hpp through oracle/_ref)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import generators as G


def same(p, r):
    for k in ("values", "row_ptr", "col_indices"):
        assert np.array_equal(getattr(p.p_upper, k), getattr(r.p_upper, k)), k
        assert np.array_equal(getattr(p.a, k), getattr(r.a, k)), k
    for k in "qlu":
        assert np.array_equal(getattr(p, k), getattr(r, k)), k


@pytest.mark.parametrize("cls", G.CLASSES)
@pytest.mark.parametrize("scale", [0, 1, 5, 7])
def test_generate_matches_reference(cls, scale):
    for seed in (0, 7):
        same(G.generate(cls, scale, seed), O.ref_generate(cls, scale, seed))


@pytest.mark.parametrize("kind,a,b,c", [("random", 100, 1000, 3), ("random", 90, 900, 13),
                                        ("lasso", 400, 4000, 0), ("huber", 300, 3000, 0),
                                        ("svm", 100, 20000, 0), ("portfolio", 4000, 40, 0),
                                        ("equality", 300, 150, 0), ("control", 30, 15, 10)])
def test_explicit_matches_reference(kind, a, b, c):
    same(G.generate_explicit(kind, a, b, c, seed=3), O.ref_generate_explicit(kind, a, b, c, seed=3))


def test_thread_count_invariance():
    p1 = G.generate("svm", 6, 2)
    G.set_threads(1)
    try:
        p2 = G.generate("svm", 6, 2)
    finally:
        G.set_threads(0)
    same(p1, p2)


def test_config1_shape():
    p = G.config("1")
    assert (p.n, p.m, p.p_upper.nnz, p.a.nnz) == (1000, 10000, 3988, 1500208)
