"""Pins for the oracle's expansion (orc_spgemm), independent of the oracle itself.

O1 pins: dense brute force on tiny inputs (numpy fp64 A@A,
boolean product for the structure), the flops definition P:173-175 counted by an
integer boolean product, the column-stochastic invariant, closed forms (identity,
K_m with loops), and scipy's sparse product as a library routine.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
import synth


def _dense(m):
    d = np.zeros((m.nrows, m.ncols))
    for j in range(m.ncols):
        a, b = int(m.colptr[j]), int(m.colptr[j + 1])
        d[m.rows[a:b], j] = m.vals[a:b]
    return d


def _pattern(m):
    d = np.zeros((m.nrows, m.ncols), dtype=np.int64)
    for j in range(m.ncols):
        a, b = int(m.colptr[j]), int(m.colptr[j + 1])
        d[m.rows[a:b], j] = 1
    return d


@pytest.mark.parametrize("seed", range(12))
def test_expand_matches_dense_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 64))
    A = synth.random_sparse(n, n, float(rng.uniform(0.02, 0.4)), seed=seed, empty_cols=0.1)
    Cm, flops = O.expand(A)
    D = _dense(O.as_mat(A))
    ref = D @ D
    P = _pattern(A)
    struct = (P @ P) > 0
    got = _dense(Cm)
    # structure: exactly the boolean product (Q13)
    assert np.array_equal(_pattern(Cm) > 0, struct)
    # rows strictly increasing inside every column
    for j in range(Cm.ncols):
        r = Cm.rows[Cm.colptr[j]:Cm.colptr[j + 1]]
        assert np.all(np.diff(r) > 0)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=0)
    # flops(AA) = number of nontrivial products a_ik*a_kj, counted by the
    # integer boolean product: sum_{i,j} #{k : a_ik != 0 and a_kj != 0}
    assert flops.sum() == int((P @ P).sum())
    assert np.array_equal(flops, (P @ P).sum(axis=0))


@pytest.mark.parametrize("seed", range(6))
def test_rectangular_spgemm_and_column_range(seed):
    rng = np.random.default_rng(100 + seed)
    m, p, n = (int(x) for x in rng.integers(1, 40, size=3))
    A = synth.random_sparse(m, p, 0.2, seed=seed)
    B = synth.random_sparse(p, n, 0.2, seed=seed + 50, empty_cols=0.2)
    b = int(rng.integers(0, n))
    e = int(rng.integers(b, n + 1))
    Cm, flops = O.spgemm(A, B, b, e)
    ref = _dense(O.as_mat(A)) @ _dense(O.as_mat(B))[:, b:e]
    np.testing.assert_allclose(_dense(Cm), ref, rtol=1e-12, atol=0)
    assert np.array_equal(_pattern(Cm) > 0, (_pattern(A) @ _pattern(B)[:, b:e]) > 0)
    assert np.array_equal(flops, (_pattern(A) @ _pattern(B)[:, b:e]).sum(axis=0))


def test_flops_spec_examples():
    # A=I3 -> flops 3, cf 1; 2x2 all-ones -> flops 8, nnz 4, cf 2
    I3 = synth.Csc(3, 3, np.arange(4, dtype=np.int64), np.arange(3, dtype=np.int32),
                   np.ones(3, np.float32))
    Cm, f = O.expand(I3)
    assert f.sum() == 3 and Cm.nnz == 3
    J2 = synth.Csc(2, 2, np.array([0, 2, 4], np.int64), np.array([0, 1, 0, 1], np.int32),
                   np.ones(4, np.float32))
    Cm, f = O.expand(J2)
    assert f.sum() == 8 and Cm.nnz == 4 and f.sum() / Cm.nnz == 2


@pytest.mark.parametrize("mm", [1, 2, 5, 17])
def test_clique_closed_form(mm):
    # unit-weight K_m with loops: A = J/m, A.A = J/m (SURVEY c.3 O1 closed form)
    G = synth.pairs_to_symmetric_csc(mm, *np.triu_indices(mm, 1), np.ones(mm * (mm - 1) // 2))
    A = O.preprocess(G)
    np.testing.assert_allclose(_dense(A), np.full((mm, mm), 1.0 / mm), rtol=1e-15)
    Cm, _ = O.expand(A)
    np.testing.assert_allclose(_dense(Cm), np.full((mm, mm), 1.0 / mm), rtol=1e-14)


def test_column_stochastic_invariant_c1():
    # sum_i (A.A)_ij = sum_k a_kj sum_i a_ik = 1 for column-stochastic A
    A = O.preprocess(synth.planted_partition())
    Cm, _ = O.expand(A)
    sums = np.add.reduceat(Cm.vals, Cm.colptr[:-1])
    np.testing.assert_allclose(sums, 1.0, atol=1e-13)


def test_scipy_library_product_c1_and_c2_sample():
    for G in (synth.planted_partition(), synth.cliques_noise().slice_cols(0, 20000)):
        A = O.preprocess(G)
        S = sp.csc_matrix((A.vals, A.rows, A.colptr), shape=(A.nrows, A.ncols))
        cols = np.arange(0, A.ncols, max(1, A.ncols // 300))
        for j in cols[:40]:
            Cm, _ = O.expand(A, int(j), int(j) + 1)
            ref = (S @ S[:, int(j)]).tocsc()
            ref.sort_indices()
            assert np.array_equal(Cm.rows, ref.indices)
            np.testing.assert_allclose(Cm.vals, ref.data, rtol=1e-12)


def test_preprocess_spec_examples():
    # [2,2] without loops -> [0.5,0.5]; empty column with loops -> single 1.0
    G = synth.Csc(3, 2, np.array([0, 2, 2], np.int64), np.array([0, 2], np.int32),
                  np.array([2.0, 2.0], np.float32))
    A = O.preprocess(G, add_loops=False)
    assert A.vals.tolist() == [0.5, 0.5]
    G = synth.Csc(2, 2, np.array([0, 0, 0], np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
    A = O.preprocess(G, add_loops=True)
    assert A.rows.tolist() == [0, 1] and A.vals.tolist() == [1.0, 1.0]
    A = O.preprocess(synth.planted_partition())
    np.testing.assert_allclose(np.add.reduceat(A.vals, A.colptr[:-1]), 1.0, atol=1e-14)
    assert np.all(np.diff(A.colptr) == np.diff(synth.planted_partition().colptr) + 1)
