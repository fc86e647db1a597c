"""Pins for the oracle's Cohen estimator (O6) and its merge / Alg. 2 stack (O7).

Cohen (§V, lambda = 1 at P:1036):
  * Philox-4x32-10 against the Random123 known-answer vectors (Salmon et al., SC'11);
  * key distribution Exp(1) (mean 1, P(X > 1) = e^-1);
  * two-layer min propagation against brute-force reachability from the boolean
    product (c[s][j] = min over all first-layer vertices reaching j);
  * unbiasedness E[(r-1)/sum] = nnz_j (Gamma(r, mu) closed form, SURVEY c.3 O6) by
    Monte-Carlo over seeds.
Merge: the merged list equals the dense sum of blocks; Alg. 2's stack depth after i
pushes is popcount(i); binary merge == multiway merge; the SUMMA block
identity sum_q A[:, K_q] A[K_q, :] == A.A.
"""
import numpy as np
import pytest

import oracle as O
import synth

# Random123 kat_vectors, philox4x32 with 10 rounds: (counter, key) -> output
KAT = [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_known_answers(ctr, key, out):
    assert O.philox(ctr, key).tolist() == out


def test_keys_are_exponential():
    A = synth.random_sparse(20000, 1, 0.0001, seed=0)
    _, X, _ = O.cohen(A, synth.random_sparse(1, 1, 1.0, seed=0), r=5, seed=7, return_keys=True)
    X = X.astype(np.float64).ravel()
    assert X.min() > 0
    assert abs(X.mean() - 1.0) < 0.02
    assert abs((X > 1.0).mean() - np.exp(-1.0)) < 0.01


@pytest.mark.parametrize("seed", range(4))
def test_min_propagation_bruteforce(seed):
    rng = np.random.default_rng(seed)
    m, p, n = (int(x) for x in rng.integers(5, 40, size=3))
    A = synth.random_sparse(m, p, 0.15, seed=seed, empty_cols=0.1)
    B = synth.random_sparse(p, n, 0.15, seed=seed + 9, empty_cols=0.1)
    r = 7
    est, X, M = O.cohen(A, B, r=r, seed=seed, return_keys=True)
    PA = np.zeros((m, p), bool)
    for k in range(p):
        PA[A.rows[A.colptr[k]:A.colptr[k + 1]], k] = True
    PB = np.zeros((p, n), bool)
    for j in range(n):
        PB[B.rows[B.colptr[j]:B.colptr[j + 1]], j] = True
    reach = (PA.astype(int) @ PB.astype(int)) > 0          # first-layer i reaches column j
    for j in range(n):
        rows = np.nonzero(reach[:, j])[0]
        if len(rows) == 0:
            assert est[j] == 0.0
            continue
        c = X[:, rows].min(axis=1).astype(np.float64)
        assert est[j] == pytest.approx((r - 1) / c.sum(), rel=1e-12)
        # keys are the Philox formula's: spot-check one against the scalar entry point
        assert X[0, rows[0]] == O.cohen_key(seed, 0, int(rows[0]))


def test_estimator_unbiased():
    # E[(r-1)/sum_s Y_s] = mu exactly for Y_s ~ Exp(mu) (Gamma(r, mu)); Monte-Carlo
    A = O.preprocess(synth.planted_partition())
    Cm, _ = O.expand(A)
    exact = np.diff(Cm.colptr).astype(np.float64)
    ests = np.stack([O.cohen(A, A, r=10, seed=s) for s in range(200)])
    mean = ests.mean(axis=0)
    rel = np.abs(mean - exact) / exact
    assert np.median(rel) < 0.05
    # total within the paper's "within 10%" range for a single seed, median
    tot = np.abs(ests.sum(axis=1) - exact.sum()) / exact.sum()
    assert np.median(tot) < 0.10


def _blocks(n, parts):
    cuts = np.linspace(0, n, parts + 1).astype(int)
    return list(zip(cuts[:-1], cuts[1:]))


def _sub(M, r0, r1, c0, c1):
    Mt = M.slice_cols(c0, c1) if hasattr(M, "slice_cols") else M
    rows, vals, cp = [], [], [0]
    for j in range(c0, c1):
        a, b = int(M.colptr[j]), int(M.colptr[j + 1])
        rr = M.rows[a:b]
        sel = (rr >= r0) & (rr < r1)
        rows.append(rr[sel] - r0)
        vals.append(M.vals[a:b][sel])
        cp.append(cp[-1] + int(sel.sum()))
    del Mt
    return O.Mat(r1 - r0, c1 - c0, np.array(cp, np.int64),
                 np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32),
                 np.concatenate(vals).astype(np.float64) if vals else np.zeros(0))


@pytest.mark.parametrize("s", [1, 2, 4, 8])
def test_summa_block_identity_and_binary_merge(s):
    A = O.preprocess(synth.planted_partition())
    n = A.ncols
    full, _ = O.expand(A)
    parts = []
    for (k0, k1) in _blocks(n, s):
        Ak = _sub(A, 0, n, k0, k1)           # A[:, K_q]
        Bk = _sub(A, k0, k1, 0, n)           # A[K_q, :]
        Pq, _ = O.spgemm(Ak, Bk)
        parts.append(Pq)
    trace = []
    mb = O.binary_merge(parts, trace)
    mw = O.merge(parts)
    assert trace == [bin(i).count("1") for i in range(1, s + 1)]
    for M in (mb, mw):
        assert np.array_equal(M.colptr, full.colptr) and np.array_equal(M.rows, full.rows)
        np.testing.assert_allclose(M.vals, full.vals, rtol=1e-12)


def test_merge_is_dense_sum():
    mats = [synth.random_sparse(30, 25, 0.2, seed=s, empty_cols=0.2) for s in range(5)]
    M = O.merge(mats)
    ref = sum(O.as_mat(m).dense() for m in mats)
    np.testing.assert_allclose(M.dense(), ref, rtol=1e-12)
    struct = sum((O.as_mat(m).dense() != 0).astype(int) for m in mats) > 0
    assert np.array_equal(M.dense() != 0, struct)
