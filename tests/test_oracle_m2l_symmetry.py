"""M2L offset symmetry used by the per-pair FFT product (k_m2l_items, which reads the spectra of the 56 offsets |o| and reflects them).

The product keeps the operator spectra of only the 158 offsets o of one half and
reads offset -o as the conjugate.  In real space that is K_{-o} = K_o^T for the
oracle's M2L matrices (upward equivalent -> downward check):
L and G are even in r and symmetric in their indices, and both surfaces of M2L
lie on the same lattice about their box centres, so swapping source and target
boxes transposes the matrix.  The DFT of a real sequence reversed in index is
the conjugate of its DFT, which is the Fourier-space form the product uses.
Also pinned: -o is offset 315 - o in the lexicographic offset table."""
import numpy as np
import pytest

from oracle.operators import Operators, v_offsets


def test_negated_offset_is_mirror_index():
    offs = v_offsets()
    assert len(offs) == 316
    for i, o in enumerate(offs):
        assert offs[315 - i] == tuple(-v for v in o)


@pytest.mark.parametrize("ml,k", [("L", 1), ("G", 3)])
def test_m2l_negated_offset_is_transpose(ml, k):
    ops = Operators(ml, 4)
    for o in [(2, 0, 0), (3, -2, 1), (-3, 3, 3), (0, 2, -2)]:
        a = ops.m2l[o]
        b = ops.m2l[tuple(-v for v in o)]
        assert a.shape == b.shape == (ops.n, ops.n)
        assert np.allclose(b, a.T, rtol=1e-13, atol=1e-13 * np.abs(a).max())


def test_reversed_real_sequence_has_conjugate_dft():
    rng = np.random.default_rng(7)
    x = rng.standard_normal((7, 7, 7))
    rev = np.roll(x[::-1, ::-1, ::-1], 1, axis=(0, 1, 2))  # x[-d mod n]
    assert np.allclose(np.fft.fftn(rev), np.conj(np.fft.fftn(x)), atol=1e-12)
