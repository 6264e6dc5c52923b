"""The real embedding of a complex Hermitian operator (hermitian.py, CPU only): S = [[A, -B], [B, A]]
has H's spectrum with every eigenvalue doubled, a valid strictly-ascending CSR layout, and maps its
eigenvectors [x; y] to H's x + iy."""
import numpy as np

import paper_2604_00914_b200 as adp
from paper_2604_00914_b200 import configs


def test_embedding_spectrum_and_layout():
    h = configs.peierls_lattice(12, phi=1.0 / 8.0, seed=2)
    s = adp.hermitian_embedding(h)
    s.validate()
    assert not s.is_complex and s.n_rows == 2 * h.n_rows
    sd = s.to_dense()
    assert np.array_equal(sd, sd.T)
    eh = np.linalg.eigvalsh(h.to_dense())
    es = np.linalg.eigvalsh(sd)
    assert np.allclose(es, np.repeat(eh, 2), atol=1e-12 * np.abs(eh).max())
    w, z = np.linalg.eigh(sd)
    n = h.n_rows
    v = z[:n, 5] + 1j * z[n:, 5]
    assert np.linalg.norm(h.to_dense() @ v - w[5] * v) <= 1e-12 * np.abs(eh).max()


def test_embedding_drops_structural_zeros():
    # a real-valued Hermitian input: the imaginary blocks vanish, S = diag(A, A)
    r, c = np.array([0, 0, 1, 1, 2]), np.array([0, 1, 0, 1, 2])
    h = adp.CsrMatrix.from_triplets(3, 3, r, c, np.array([2.0, 1.0, 1.0, 3.0, 4.0], np.complex128))
    s = adp.hermitian_embedding(h)
    assert s.nnz == 2 * h.nnz
    assert np.array_equal(s.to_dense(), np.kron(np.eye(2), h.to_dense().real))
