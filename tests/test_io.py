"""The I/O around the kernel: mcl_graph_read / mcl_clusters_write in
libmclx.so, host-side (runs without a GPU).  Pins: SPEC S:547-559's examples, scipy's
MatrixMarket reader on random files, the symmetrisation identity max(A, A^T), and the
cluster-file format on two disjoint triangles."""
import os

import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp

import synth

M = pytest.importorskip("paper_2002_10083_b200", reason="libmclx.so not built")


def write(tmp_path, name, text):
    p = os.path.join(tmp_path, name)
    with open(p, "w") as f:
        f.write(text)
    return p


def dense(g):
    d = np.zeros((g.nrows, g.ncols))
    for j in range(g.ncols):
        for q in range(g.colptr[j], g.colptr[j + 1]):
            d[g.rows[q], j] += g.vals[q]
    return d


def test_spec_examples(tmp_path):
    # 3-vertex triangle MatrixMarket -> 3 x 3, nnz 6 after the symmetric expansion
    p = write(tmp_path, "tri.mtx", "%%MatrixMarket matrix coordinate real symmetric\n"
              "% a comment\n3 3 3\n2 1 0.5\n3 1 1.5\n3 2 2.0\n")
    g = M.read_graph(p, symmetrize=False)
    assert (g.ncols, g.nnz) == (3, 6) and g.labels is None
    assert np.array_equal(dense(g), [[0, .5, 1.5], [.5, 0, 2], [1.5, 2, 0]])
    # TSV "a b 1.0 / b c 2.0" -> 3 x 3 with 2 nonzeros and a label map of size 3
    p = write(tmp_path, "e.tsv", "a\tb\t1.0\nb\tc\t2.0\n")
    g = M.read_graph(p, symmetrize=False)
    assert (g.ncols, g.nnz, g.labels) == (3, 2, ["a", "b", "c"])
    assert dense(g)[1, 0] == 1.0 and dense(g)[2, 1] == 2.0
    # pattern MatrixMarket -> all values 1.0
    p = write(tmp_path, "p.mtx", "%%MatrixMarket matrix coordinate pattern general\n2 2 3\n1 1\n2 1\n1 2\n")
    g = M.read_graph(p, symmetrize=False)
    assert g.nnz == 3 and np.all(g.vals == 1.0)


def test_duplicates_summed_zeros_dropped(tmp_path):
    p = write(tmp_path, "d.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 4\n"
              "1 1 2.0\n1 1 -0.0\n2 1 1.0\n2 1 2.5\n")
    g = M.read_graph(p, symmetrize=False)
    assert np.array_equal(dense(g), [[2.0, 0], [3.5, 0]])
    p = write(tmp_path, "z.tsv", "x y 0\n")  # an exact-zero edge is dropped, its labels kept
    g = M.read_graph(p, symmetrize=False)
    assert g.ncols == 2 and g.nnz == 0


@pytest.mark.parametrize("text,msg", [
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", ":3: malformed entry"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n", "above the diagonal"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 -1.0\n", "negative"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "outside"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "declares 2"),
    ("%%MatrixMarket matrix array real general\n2 2\n", "unsupported"),
    ("a b 1\nc\n", ":2: expected"),
    ("a b -2\n", "negative"),
])
def test_errors_name_the_line(tmp_path, text, msg):
    p = write(tmp_path, "bad.txt", text)
    with pytest.raises(M.MclError) as e:
        M.read_graph(p)
    assert msg in str(e.value) and e.value.code == -3


def test_non_square_and_missing(tmp_path):
    p = write(tmp_path, "r.mtx", "%%MatrixMarket matrix coordinate real general\n2 3 0\n")
    with pytest.raises(M.MclError) as e:
        M.read_graph(p)
    assert e.value.code == -2
    with pytest.raises(M.MclError):
        M.read_graph(os.path.join(tmp_path, "nope.mtx"))


@pytest.mark.parametrize("seed", range(3))
def test_matches_scipy_mmread(tmp_path, seed):
    """A random general MatrixMarket file reads to the same matrix as scipy.io.mmread (an
    independent parser), and symmetrize gives max(A, A^T)."""
    A = sp.random(60, 60, density=0.05, random_state=seed, format="coo", dtype=np.float64)
    A.data = np.round(A.data * 100 + 1) / 8  # exactly representable in fp32
    p = os.path.join(tmp_path, "r.mtx")
    scipy.io.mmwrite(p, A)
    ref = scipy.io.mmread(p).toarray()
    g = M.read_graph(p, symmetrize=False)
    assert np.array_equal(dense(g), ref)
    assert all(np.all(np.diff(g.rows[g.colptr[j]:g.colptr[j + 1]]) > 0) for j in range(60))
    gs = M.read_graph(p, symmetrize=True)
    assert np.array_equal(dense(gs), np.maximum(ref, ref.T))


def test_symmetrize_idempotent_on_synth(tmp_path):
    """A symmetric generator graph written as a general edge list reads back unchanged."""
    G = synth.planted_partition()
    p = os.path.join(tmp_path, "c1.tsv")
    with open(p, "w") as f:
        for j in range(G.ncols):
            for q in range(G.colptr[j], G.colptr[j + 1]):
                f.write(f"v{j}\tv{G.rows[q]}\t{float(G.vals[q])!r}\n")
    g = M.read_graph(p, symmetrize=True)
    ids = np.array([int(s[1:]) for s in g.labels])
    d = dense(g)
    ref = np.zeros((G.ncols, G.ncols))
    for j in range(G.ncols):
        for q in range(G.colptr[j], G.colptr[j + 1]):
            ref[G.rows[q], j] = G.vals[q]
    assert np.array_equal(d, ref[np.ix_(ids, ids)].astype(np.float32))


def test_clusters_file(tmp_path):
    """Two disjoint triangles -> exactly 2 lines, members ascending, labels used."""
    p = os.path.join(tmp_path, "c.txt")
    M.write_clusters(p, np.array([0, 0, 0, 1, 1, 1], np.int32))
    assert open(p).read() == "1 2 3\n4 5 6\n"
    g = M.HostGraph(4, 4, np.zeros(5, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32),
                    ["w", "x", "y", "z"])
    M.write_clusters(p, np.array([0, 1, 0, 1], np.int32), g)
    assert open(p).read() == "w y\nx z\n"


@pytest.mark.gpu
def test_cli_end_to_end_matches_oracle(tmp_path):
    """python -m paper_2002_10083_b200 GRAPH OUT on C1 written as a symmetric MatrixMarket file:
    the cluster file lists the oracle's clusters (canonical order, 1-based ids)."""
    import subprocess
    import sys

    import oracle as O
    G = synth.planted_partition()
    p = os.path.join(tmp_path, "c1.mtx")
    with open(p, "w") as f:
        lower = [(int(G.rows[q]), j, float(G.vals[q])) for j in range(G.ncols)
                 for q in range(G.colptr[j], G.colptr[j + 1]) if G.rows[q] >= j]
        f.write(f"%%MatrixMarket matrix coordinate real symmetric\n{G.nrows} {G.ncols} {len(lower)}\n")
        for i, j, w in lower:
            f.write(f"{i + 1} {j + 1} {w!r}\n")
    out = os.path.join(tmp_path, "clusters.txt")
    r = subprocess.run([sys.executable, "-m", "paper_2002_10083_b200", p, out], capture_output=True,
                       text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr
    ref = O.mcl(G)
    lines = []
    for c in range(ref.nclusters):
        lines.append(" ".join(str(i + 1) for i in np.nonzero(ref.labels == c)[0]))
    assert open(out).read() == "\n".join(lines) + "\n"
