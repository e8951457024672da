"""Host-side proofs for the arithmetic the fused compress kernel relies on (no GPU).

tools/exactness_bounds.py models the kernel's fp32 inverse (the transposed 22-addition graph, columns
then rows, in the kernel's operation order) on affine forms of the 64 pixels of a block.  Here the
model's outputs are compared, as exact integer forms, with plain matrix algebra written out in the
test, for every r:

* direct   (kernel rows that compute e = 576 x - R):  graph output == T^T (W . M_r . Y) T  (+ DC bias)
* residual (kernel for r >= ADCT_RESID_FROM):          graph output == 576 x - T^T (W . M_r . Y) T,
  i.e. C0^T (W . (1 - M_r) . Y) C0 = 576 x - R, which rests on r = 64 being lossless (pin P8)

and every intermediate node stays below 2^24 in magnitude, so fp32 evaluates it exactly.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import exactness_bounds as EB  # noqa: E402


def _affine_R(r):
    """R = T^T (W . M_r . Y) T with Y = T X T^T, as a (64 outputs) x (64 pixels) integer matrix."""
    T, W = EB.T, EB.W
    M = np.array([[EB.zz(i, j) < r for j in range(8)] for i in range(8)])
    G = np.zeros((64, 64), dtype=np.int64)
    for p in range(64):  # impulse response of pixel p
        X = np.zeros((8, 8), dtype=np.int64)
        X[p // 8, p % 8] = 1
        Y = T @ X @ T.T
        G[:, p] = (T.T @ (W * M * Y) @ T).reshape(64)
    return G


def _forms(out):
    """graph outputs out[i][n] (affine forms) -> (64 x 64 coefficient matrix, 64 constants)"""
    A = np.zeros((64, 64), dtype=np.int64)
    c = np.zeros(64, dtype=np.int64)
    for i in range(8):
        for n in range(8):
            f = out[i][n]
            if f is not None:
                A[i * 8 + n] = f[:64]
                c[i * 8 + n] = f[64]
    return A, c


@pytest.mark.parametrize("graph", list(EB.GRAPHS))
@pytest.mark.parametrize("r", list(range(1, 65)))
def test_direct_graph_is_R(r, graph):
    """Every inverse flavour the kernels use (f32x2 inv8, one-instruction-butterfly inv8s, and the
    hybrid of the two) computes exactly T^T (W . M_r . Y) T (+ the DC bias) with every node < 2^24."""
    for bias in EB.DC_BIASES:
        m, out = EB.run(r, "direct", bias, graph)
        A, c = _forms(out)
        assert np.array_equal(A, _affine_R(r))
        assert np.all(c == bias)
        assert m < 2 ** 24


@pytest.mark.parametrize("graph", list(EB.GRAPHS))
@pytest.mark.parametrize("r", list(range(1, 64)))
def test_residual_graph_is_error(r, graph):
    m, out = EB.run(r, "residual", 0, graph)
    A, c = _forms(out)
    assert np.array_equal(A, 576 * np.eye(64, dtype=np.int64) - _affine_R(r))
    assert np.all(c == 0)
    assert m < 2 ** 24


def test_r64_lossless_identity():
    # the identity the residual form rests on: T^T (W . Y) T = 576 X for every block (P8)
    assert np.array_equal(_affine_R(64), 576 * np.eye(64, dtype=np.int64))


def test_exactness_tool_exit_code():
    assert EB.main() == 0


@pytest.mark.parametrize("row_graph", ["inv8", "inv8s"])
def test_band_chain_equals_error_per_r(row_graph):
    # k_compress_sweep_inc: after band b the running per-pixel form is 576 x - R_r, r = (b+1)(b+2)/2
    m, finals = EB.run_band_chain(getattr(EB, row_graph))
    assert m < 2 ** 24
    for r, e in finals.items():
        A_, c = _forms(e)
        assert np.array_equal(A_, 576 * np.eye(64, dtype=np.int64) - _affine_R(r)), r
        assert np.all(c == 0)


@pytest.mark.parametrize("L", list(range(8)))
def test_fully_discarded_column_identity(L):
    # compress_resid_hc: a column whose coefficients the mask discards entirely contributes
    # C0^T diag(W[:, L]) C0 H[:, L] = (576 / d_L) H[:, L] to the column pass (H = row pass of the pixels)
    T, W = EB.T, EB.W
    d = np.diag(T @ T.T)
    assert np.array_equal(T.T @ np.diag(W[:, L]) @ T, (576 // d[L]) * np.eye(8, dtype=np.int64))
    assert 576 % d[L] == 0


@pytest.mark.parametrize("L", list(range(1, 8)))
def test_row0_only_column_identity(L):
    """compress_resid_hc's partial injection (pcol_mask): for a column L >= 1 whose only kept
    coefficient is (0, L), the column inverse of the discarded rows 1..7 equals
    (576 / d_L) H - W_0L (sum_i H_i) 1 = W_0L (8 H - (sum_i H_i) 1), with W_0L = 576 / (8 d_L) an
    integer, and 8 H_i - sum_j H_j stays inside int16 for every uint8 row-pass column."""
    T, W = EB.T, EB.W
    d = np.diag(T @ T.T)
    D1 = np.diag(W[:, L] * (np.arange(8) != 0))           # discarded rows 1..7 of column L
    lhs = T.T @ D1 @ T
    rhs = (576 // d[L]) * np.eye(8, dtype=np.int64) - W[0, L] * np.ones((8, 8), dtype=np.int64)
    assert np.array_equal(lhs, rhs)
    assert W[0, L] * 8 == 576 // d[L]
    # H[:, L] = (X T^T)[:, L] = X T[L]: |8 H_i - sum_j H_j| <= 14 max|H| over uint8 rows
    assert 14 * (255 * max(T[L][T[L] > 0].sum(), -T[L][T[L] < 0].sum())) < 2 ** 15


@pytest.mark.parametrize("L", list(range(1, 8)))
def test_rows01_only_column_identity(L):
    """compress_resid_hc's {0, 1}-kept injection (p2col_mask): for a column whose kept set is
    {(0, L), (1, L)}, the discarded rows' column inverse is W_0L (8 H - (sum_i H_i) 1) -
    W_1L (sum_i T1_i H_i) T1 with integer W_0L, W_1L, and sum_i T1_i H_i stays inside int16."""
    T, W = EB.T, EB.W
    d = np.diag(T @ T.T)
    D = np.diag(W[:, L] * (np.arange(8) >= 2))            # discarded rows 2..7 of column L
    lhs = T.T @ D @ T
    one = np.ones(8, dtype=np.int64)
    rhs = W[0, L] * (8 * np.eye(8, dtype=np.int64) - np.outer(one, one)) - W[1, L] * np.outer(T[1], T[1])
    assert np.array_equal(lhs, rhs)
    assert 576 // d[L] == 8 * W[0, L] and W[1, L] * 6 * d[L] == 576
    assert 6 * 255 * max(T[L][T[L] > 0].sum(), -T[L][T[L] < 0].sum()) < 2 ** 15


@pytest.mark.parametrize("r", list(range(23, 64)))
def test_pcol_columns_are_the_row0_only_ones(r):
    M = np.array([[EB.zz(i, j) < r for j in range(8)] for i in range(8)])
    want = [L for L in range(1, 8) if M[0, L] and not M[1:, L].any()]
    # triangular r = (s+1)(s+2)/2 leave column s with (0, s) alone: r = 28 -> 6, r = 36 -> 7
    if r == 28:
        assert want == [6]
    if r == 36:
        assert want == [7]


@pytest.mark.parametrize("r", list(range(1, 64)))
def test_hcol_columns_are_exactly_the_empty_ones(r):
    # the kernel injects column L iff no zig-zag index < r lies in it (hcol_mask)
    M = np.array([[EB.zz(i, j) < r for j in range(8)] for i in range(8)])
    empty = [L for L in range(8) if not M[:, L].any()]
    # for the residual kernels (r >= 24) these are the columns 7 (r <= 28) and 6 (r <= 27)
    if r >= 24:
        assert empty == [L for L in (6, 7) if (L == 7 and r <= 28) or (L == 6 and r <= 27)]
