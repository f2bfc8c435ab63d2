"""MatrixMarket I/O (proj/src/testmat.cpp:134-355) and the CSR handle's validation
(proj/src/matrix.cpp:79-104), host side; the device densification is in test_gpu_engine."""
import numpy as np
import pytest

from paper_2509_21963_b200 import MatrixHandle
from paper_2509_21963_b200.mmio import read_matrix_market, write_matrix_market


def test_dense_round_trip(tmp_path):
    a = np.random.default_rng(1).standard_normal((7, 5))
    p = tmp_path / "a.mtx"
    write_matrix_market(str(p), MatrixHandle.dense(a))
    b = read_matrix_market(str(p))
    assert not b.is_sparse and np.array_equal(b.to_numpy(), a)  # %.17g round-trips exactly


def test_sparse_round_trip_and_symmetric(tmp_path):
    h = MatrixHandle.sparse_csr(3, 4, [0, 2, 2, 3], [0, 3, 1], [1.5, -2.0, 7.0])
    p = tmp_path / "s.mtx"
    write_matrix_market(str(p), h)
    g = read_matrix_market(str(p))
    assert g.is_sparse and g.nnz == 3 and np.array_equal(g.to_numpy(), h.to_numpy())
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n% comment\n\n3 3 2\n2 1 4\n3 3 5\n")
    s = read_matrix_market(str(p)).to_numpy()
    assert s[1, 0] == 4 and s[0, 1] == 4 and s[2, 2] == 5
    p.write_text("%%MatrixMarket matrix array real symmetric\n2 2\n1\n2\n3\n")
    assert np.array_equal(read_matrix_market(str(p)).to_numpy(), [[1, 2], [2, 3]])


@pytest.mark.parametrize("body,msg", [
    ("", "empty file"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1\n", "unsupported field"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 2\n", "duplicate entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", "out of range"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n", "file ended after 1"),
    ("%%MatrixMarket matrix array real general\n2 2\n1 2 3\n", "expected 4 values"),
    ("%%MatrixMarket matrix array real general\n1 1\nnan\n", "non-finite"),
    ("%%MatrixMarket matrix array real general\n1 1\n1x\n", "malformed numeric"),
])
def test_parse_errors(tmp_path, body, msg):
    p = tmp_path / "bad.mtx"
    p.write_text(body)
    with pytest.raises(RuntimeError, match=msg):
        read_matrix_market(str(p))


def test_csr_validation():
    with pytest.raises(ValueError, match="rows\\+1"):
        MatrixHandle.sparse_csr(2, 2, [0, 1], [0], [1.0])
    with pytest.raises(ValueError, match="strictly increasing"):
        MatrixHandle.sparse_csr(1, 3, [0, 2], [2, 1], [1.0, 2.0])
    with pytest.raises(IndexError):
        MatrixHandle.sparse_csr(1, 2, [0, 1], [5], [1.0])
    with pytest.raises(ValueError, match="non-finite"):
        MatrixHandle.sparse_csr(1, 1, [0, 1], [0], [np.inf])
