"""CPU audit of the quantiser decision the QUANT kernels take (reading R10).

The kernel decides k = round-to-nearest(Y * c') in one fp32 FMA (exact product, one rounding to an
integer via the 1.5*2^23 magic constant), with c' = adct_quant_reciprocals(q) from the library's
host code.  This test (no GPU needed) checks, against the oracle's exact rational decision:
  * c' is the smallest fp32 strictly above 1/(q sqrt(d_k d_l))   (checked with Fractions);
  * for q = 16 (BASELINE C4) the decision equals round_half_away(Z/q) for EVERY reachable
    Y in [-16320, 16320] at every one of the 64 positions;
  * no product Y c' is itself an exact tie (so the FMA's round-to-nearest-even never decides).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import paper_1402_6034_b200 as A

D = [8, 6, 4, 6, 8, 6, 4, 6]
Y_ALL = np.arange(-16320, 16321, dtype=np.int64)


def kernel_decision(Y, c):
    """round-to-nearest-even of the exact product Y * c (what the FMA with the magic constant does)."""
    v = Y.astype(np.float64) * np.float64(c)       # exact: 15-bit * 24-bit significands
    assert np.all(np.abs(v - np.floor(v)) != 0.5)   # never an exact tie
    return np.rint(v).astype(np.int64)


@pytest.mark.parametrize("q", [16.0, 5.0, 3.0, 12.0, 100.0])
def test_reciprocals_are_smallest_float_above_exact(q):
    c = A.quant_reciprocals(q)
    for k in range(8):
        for l in range(8):
            dd = D[k] * D[l]
            cf = np.float32(c[k, l])
            above = lambda x: (Fraction(float(x)) * Fraction(q)) ** 2 * dd > 1
            assert above(cf)
            assert not above(np.nextafter(cf, np.float32(0)))


@pytest.mark.parametrize("q", [16.0, 5.0, 3.0])
def test_decision_equals_exact_round_half_away_on_full_domain(q):
    c = A.quant_reciprocals(q)
    for k in range(8):
        for l in range(8):
            Y = np.zeros((len(Y_ALL), 8, 8), dtype=np.int64)
            Y[:, k, l] = Y_ALL
            exact = O.to_blocks(O.quantize_exact(O.from_blocks(Y[:, None, None]), q))[:, 0, 0, k, l]
            got = kernel_decision(Y_ALL, c[k, l])
            assert np.array_equal(got, exact), (q, k, l, np.flatnonzero(got != exact)[:5])


def test_ties_exist_and_round_away():
    """The domain does contain exact ties (dd = 16, 36, 64); the decision sends them away from 0."""
    c = A.quant_reciprocals(16.0)
    # (0,0): Z/q = Y/128 -> ties at Y = 64 (mod 128); (1,1): Y/96 -> ties at Y = 48 (mod 96)
    for (k, l, y, want) in [(0, 0, 64, 1), (0, 0, -64, -1), (0, 0, 192, 2), (1, 1, 48, 1), (1, 1, -144, -2),
                            (2, 2, -32, -1)]:
        assert kernel_decision(np.array([y]), c[k, l])[0] == want


def test_reciprocals_validation():
    with pytest.raises(A.AdctError):
        A.quant_reciprocals(0.0)
    with pytest.raises(A.AdctError):
        A.quant_reciprocals(-2.0)
    with pytest.raises(A.AdctError):
        A.quant_reciprocals(float("nan"))
