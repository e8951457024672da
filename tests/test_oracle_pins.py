"""Pins for the CPU oracle (-m "not gpu"): each checks the oracle against something other
than itself — values the paper prints (tests/golden/), closed forms, invariants, brute force.
Pin numbers P1..P18 follow DESIGN.md §3 / SURVEY.md §8(c).
"""
import math

import numpy as np
import pytest

import oracle as O
from synth import images as S
from golden_io import read_golden
from reference_butterfly import Counter, forward8, inverse8

rng = np.random.default_rng(1234)


def golden_c0():
    return np.array([[int(v) for v in row] for row in read_golden("c0_matrix.txt")])


# ---------------------------------------------------------------- matrices (P1-P5, P16)

def test_P1_c0_equals_displayed_matrix():
    T = O.c0_matrix()
    assert T.shape == (8, 8)
    assert np.array_equal(T, golden_c0())
    assert set(np.unique(T)) <= {-1, 0, 1}


def test_round_half_away_matlab_convention():
    assert O.round_half_away(0.5) == 1 and O.round_half_away(-0.5) == -1
    assert O.round_half_away(2.5) == 3 and O.round_half_away(-2.5) == -3
    assert O.round_half_away(1.49999) == 1
    # no entry of 2C is near a tie (reading R2 is therefore moot for C0)
    frac = np.abs(2 * O.dct_matrix()) % 1.0
    assert np.min(np.abs(frac - 0.5)) > 0.05


def test_P2_orthogonalizer_is_printed_diagonal():
    T = O.c0_matrix()
    G = T @ T.T
    assert np.array_equal(G, np.diag([8, 6, 4, 6, 8, 6, 4, 6]))
    expr = [row[0] for row in read_golden("s_diagonal.txt")]
    printed = np.array([eval(e, {"sqrt": math.sqrt}) for e in expr])
    S_ = O.orthogonalizer()
    assert np.allclose(S_, np.diag(printed), atol=1e-14)


def test_P3_proposed_is_orthogonal():
    C = O.proposed_matrix()
    assert np.abs(C @ C.T - np.eye(8)).max() <= 1e-12        # P:228 "(i) it is orthogonal"
    assert np.abs(C.T @ C - np.eye(8)).max() <= 1e-12


def test_c0_is_not_orthogonal_and_coarse():
    T = O.c0_matrix().astype(float)
    assert np.abs(np.linalg.inv(T) - T.T).max() > 0.5        # P:180-181 C0^-1 != C0^T
    # P:160-164 "C_hat = 1/2 C0", pinned against the displayed C0 (golden), not the oracle's own C0
    assert np.array_equal(2.0 * O.coarse_matrix(), golden_c0().astype(float))
    # and its rows all have the same norm only where C0's rows do: ||row||^2 = d / 4
    assert np.allclose((O.coarse_matrix() ** 2).sum(axis=1), np.array([8, 6, 4, 6, 8, 6, 4, 6]) / 4.0)


def _det_exact(M):
    """Exact integer determinant (fraction-free Bareiss elimination, Python ints)."""
    A_ = [[int(v) for v in row] for row in M]
    n, sign, prev = len(A_), 1, 1
    for k in range(n - 1):
        if A_[k][k] == 0:
            sw = next((i for i in range(k + 1, n) if A_[i][k] != 0), None)
            if sw is None:
                return 0
            A_[k], A_[sw] = A_[sw], A_[k]
            sign = -sign
        for i in range(k + 1, n):
            for j in range(k + 1, n):
                A_[i][j] = (A_[i][j] * A_[k][k] - A_[i][k] * A_[k][j]) // prev
        prev = A_[k][k]
    return sign * A_[n - 1][n - 1]


def test_F4_roundoff_family_pins():
    """F4 ("floor and ceiling functions can be considered instead of the round-off
    function"): the generic f(2 C) builder reproduces the printed C0 for f = round (and its polar
    factor the printed S . C0); floor(2 C) is singular (its DC row 2/(2 sqrt 2) < 1 floors to 0), so it
    has no orthogonalisation; ceil(2 C) has entries in {0, 1}, exact determinant 16 (Bareiss, no
    floating point), a non-diagonal Gram matrix, and its polar factor is orthogonal with
    S = (T T^T)^(-1/2) symmetric positive definite."""
    assert np.array_equal(O.roundoff_matrix("round"), golden_c0())
    assert np.allclose(O.polar_orthogonal(golden_c0()), O.proposed_matrix(), atol=1e-14)
    Tf = O.roundoff_matrix("floor")
    assert np.all(Tf[0] == 0) and _det_exact(Tf) == 0
    with pytest.raises(Exception):
        O.polar_orthogonal(Tf)
    Tc = O.roundoff_matrix("ceil")
    assert set(np.unique(Tc)) <= {0, 1}
    assert _det_exact(Tc) == 16
    G = Tc @ Tc.T
    assert np.any(G - np.diag(np.diag(G)) != 0)
    Cc = O.ceil_matrix()
    assert np.abs(Cc @ Cc.T - np.eye(8)).max() <= 1e-12
    S_ = O.orthogonalizer(Tc)
    assert np.allclose(S_, S_.T, atol=1e-14) and np.all(np.linalg.eigvalsh(S_) > 0)
    assert np.abs(S_ @ S_ @ G.astype(float) - np.eye(8)).max() <= 1e-12
    # the polar factor is the closest orthogonal matrix to T (Frobenius): no random
    # orthogonal matrix Q may come closer
    g = np.random.default_rng(5)
    for _ in range(200):
        Q, _ = np.linalg.qr(g.normal(size=(8, 8)))
        assert np.linalg.norm(Tc - Q) >= np.linalg.norm(Tc - Cc) - 1e-12


def test_F1_sdct_sign_matrix_and_24_add_graph():
    """SDCT comparator (Table 1 P:288-289 "24 additions"): sign(C) has entries +-1 only (no
    entry of C is near 0), equals sdct_matrix() * 2 sqrt 2, and the host model of its fast graph
    equals sign(C) . x (and the transposed graph sign(C)^T . X) on unit and random vectors with
    exactly Table 1's 24 additions and no multiplications or shifts."""
    from reference_butterfly import sdct_forward8, sdct_inverse8
    T = O.sdct_sign_matrix()
    assert set(np.unique(T)) == {-1, 1} and np.abs(O.dct_matrix()).min() > 0.09
    assert np.allclose(T / (2 * math.sqrt(2)), O.sdct_matrix(), atol=1e-15)
    want = [int(v) for v in read_golden("table1_sdct.txt")[0]]
    vecs = [np.eye(8, dtype=np.int64)[i] for i in range(8)] + [rng.integers(-300, 300, 8) for _ in range(2000)]
    for v in vecs:
        k = Counter()
        assert np.array_equal(np.array(sdct_forward8(list(v), k)), T @ v)
        assert [k.adds, k.mults, k.shifts, k.adds + k.mults + k.shifts] == want
        k = Counter()
        assert np.array_equal(np.array(sdct_inverse8(list(v), k)), T.T @ v)
        assert k.adds == 24


def test_P4_frobenius_scale_0_3922():
    printed = float(read_golden("frobenius_scale.txt")[0][0])
    a = O.frobenius_optimal_scale()
    assert round(a, 4) == printed
    # independent check: 1-D minimisation of ||a C0 - C||_F by golden-section search
    C, T = O.dct_matrix(), O.c0_matrix().astype(float)
    f = lambda s: np.linalg.norm(s * T - C)
    lo, hi = 0.0, 1.0
    g = (math.sqrt(5) - 1) / 2
    for _ in range(200):
        m1, m2 = hi - g * (hi - lo), lo + g * (hi - lo)
        if f(m1) < f(m2):
            hi = m2
        else:
            lo = m1
    assert abs((lo + hi) / 2 - a) < 1e-8


def test_P5_table2_error_energy():
    rows = read_golden("table2_error_energy.txt")
    tab = {r[0]: [float(v) for v in r[1:]] for r in rows}
    eps_p = O.transfer_error_energy(O.proposed_matrix())
    eps_s = O.transfer_error_energy(O.sdct_matrix())
    for m in (1, 2, 3, 5, 6, 7):
        assert abs(eps_p[m] - tab[str(m)][3]) <= 0.01, (m, eps_p[m])   # Proposed column
        assert abs(eps_s[m] - tab[str(m)][2]) <= 0.01, (m, eps_s[m])   # SDCT column
    assert abs(eps_p[[1, 2, 3, 5, 6, 7]].sum() - tab["total"][3]) <= 0.03
    assert abs(eps_s[[1, 2, 3, 5, 6, 7]].sum() - tab["total"][2]) <= 0.03
    # m = 0, 4: transfer functions equal the DCT's
    assert eps_p[0] < 1e-12 and eps_p[4] < 1e-12


def test_P16_example_values():
    assert abs(O.dct_matrix()[1, 0] - 0.5 * math.cos(math.pi / 16)) < 1e-15
    assert round(O.dct_matrix()[1, 0], 6) == 0.490393
    assert round(O.proposed_matrix()[1, 0], 6) == round(1 / math.sqrt(6), 6) == 0.408248
    assert abs(O.psnr(1.0, 1) - 20 * math.log10(255)) < 1e-12
    assert round(float(O.psnr(1.0, 1)), 4) == 48.1308
    assert O.psnr(0.0, 64) == np.inf


# ---------------------------------------------------------------- fast algorithm (P6)

def test_P6_butterfly_equals_matrix_and_counts_22():
    T = O.c0_matrix()
    table1 = [int(v) for v in read_golden("table1_proposed.txt")[0]]
    for e in np.eye(8, dtype=np.int64):
        assert list(forward8(list(e), Counter())) == list(T @ e)
        assert list(inverse8(list(e), Counter())) == list(T.T @ e)
    for _ in range(10000):
        x = rng.integers(-255, 256, size=8)
        assert list(forward8(list(x), Counter())) == list(T @ x)
        assert list(inverse8(list(x), Counter())) == list(T.T @ x)
    k = Counter()
    forward8(list(range(8)), k)
    assert [k.adds, k.mults, k.shifts, k.adds + k.mults + k.shifts] == table1
    k = Counter()
    inverse8(list(range(8)), k)
    assert k.adds == 22 and k.mults == 0 and k.shifts == 0


# ---------------------------------------------------------------- zig-zag (P12)

def test_P12_zigzag_matches_standard_table():
    tab = np.array([[int(v) for v in row] for row in read_golden("jpeg_zigzag.txt")])
    Z = O.zigzag_index()
    assert np.array_equal(Z, tab)
    assert sorted(Z.ravel().tolist()) == list(range(64))
    assert O.zigzag_order()[:6] == [(0, 0), (0, 1), (1, 0), (2, 0), (1, 1), (0, 2)]
    assert Z[0].tolist() == [0, 1, 5, 6, 14, 15, 27, 28]
    kept5 = {tuple(c) for c in np.argwhere(O.zonal_mask(5))}
    assert kept5 == {(0, 0), (0, 1), (1, 0), (2, 0), (1, 1)}
    for r, s in [(1, 0), (3, 1), (6, 2), (10, 3), (15, 4), (21, 5), (28, 6), (36, 7)]:
        M = O.zonal_mask(r)
        ii, jj = np.indices((8, 8))
        assert np.array_equal(M, ii + jj <= s)               # triangular r <-> full anti-diagonals
        assert np.array_equal(M, M.T)
    with pytest.raises(ValueError):
        O.zonal_mask(0)
    with pytest.raises(ValueError):
        O.zonal_mask(65)


# ---------------------------------------------------------------- 2-D transform

def brute_forward(X, T):
    """Y[k][l] = sum_a sum_b T[k][a] X[a][b] T[l][b] with Python loops."""
    return [[sum(T[k][a] * X[a][b] * T[l][b] for a in range(8) for b in range(8))
             for l in range(8)] for k in range(8)]


def test_forward_int_brute_force_and_layout():
    T = O.c0_matrix().tolist()
    img = rng.integers(0, 256, size=(16, 24), dtype=np.uint8)
    Y = O.forward_int(img)[0]
    for by in range(2):
        for bx in range(3):
            X = img[8 * by:8 * by + 8, 8 * bx:8 * bx + 8].astype(int).tolist()
            assert Y[8 * by:8 * by + 8, 8 * bx:8 * bx + 8].tolist() == brute_forward(X, T)


def test_P11_range_extremes_and_constant_blocks():
    full = np.full((8, 8), 255, dtype=np.uint8)
    Y = O.forward_int(full)[0]
    assert Y[0, 0] == 16320 and np.count_nonzero(Y) == 1
    for v in (0, 1, 77, 255):
        img = np.full((16, 16), v, dtype=np.uint8)
        assert np.abs(O.reconstruct_zonal(img, 1) - v).max() < 1e-12   # r = 1 lossless on constants
    # checkerboards / random extremes stay inside the statically derived int16 range
    for _ in range(200):
        X = rng.choice([0, 255], size=(8, 8)).astype(np.uint8)
        Y = O.forward_int(X)
        assert Y.min() >= -8160 and Y.max() <= 16320


def test_P13_literal_float_vs_exact_integer():
    img = S.corpus_c2(3, 64, 64)
    Z = O.forward_scaled(img)
    Y = O.forward_int(img)
    d = np.array([8, 6, 4, 6, 8, 6, 4, 6], dtype=float)
    scale = np.tile(1 / np.sqrt(np.outer(d, d)), (8, 8))
    assert np.abs(Z - Y * scale).max() <= 1e-12 * max(1.0, np.abs(Z).max())


def test_P7_dc_rows_equal_dct_and_r1_equals_dct():
    C, Cd = O.proposed_matrix(), O.dct_matrix()
    assert np.abs(C[[0, 4]] - Cd[[0, 4]]).max() < 1e-15
    img = S.corpus_c2(3, 64, 64)
    sp = O.compress_zonal_sse(img, 1)
    sd = O.compress_zonal_sse(img, 1, Cd)
    assert np.allclose(sp, sd, rtol=1e-12)
    Zp, Zd = O.forward_scaled(img), O.forward_scaled(img, Cd)
    B1, B2 = O.to_blocks(Zp), O.to_blocks(Zd)
    for (i, j) in [(0, 0), (0, 4), (4, 0), (4, 4)]:
        assert np.abs(B1[..., i, j] - B2[..., i, j]).max() < 1e-9


def test_P8_r64_is_lossless():
    img = S.corpus_c2(3, 64, 64)
    rec = O.reconstruct_zonal(img, 64)
    assert np.abs(rec - img).max() < 1e-9
    R = O.reconstruct_zonal_exact(img, 64)
    assert np.array_equal(R, 576 * img.astype(np.int64))
    assert np.all(O.psnr(O.sse_per_image(img, np.rint(rec)), 64 * 64) == np.inf)


def test_P9_parseval_exact_integer_identity():
    img = S.corpus_c2(3, 64, 64)
    d = np.array([8, 6, 4, 6, 8, 6, 4, 6])
    W = 576 // np.outer(d, d)
    Y = O.to_blocks(O.forward_int(img))
    x = img.astype(np.int64)
    for r in (1, 5, 10, 17, 36, 63, 64):
        R = O.reconstruct_zonal_exact(img, r)
        sse576 = O.compress_zonal_sse576(img, r)
        kept = (W * O.zonal_mask(r) * Y * Y).reshape(3, -1).sum(1)
        assert np.array_equal(sse576, 576 * (576 * (x * x).reshape(3, -1).sum(1) - kept))
        sse = O.compress_zonal_sse(img, r)
        assert np.allclose(sse, sse576 / 576.0 ** 2, rtol=1e-10, atol=1e-9)
        rec = O.reconstruct_zonal(img, r)
        assert np.abs(rec - R / 576.0).max() < 1e-10


def test_P9b_sse576_dc_only_closed_form_and_lossless():
    # r = 1 keeps only the DC: every pixel of a block reconstructs to the block mean, so
    # 576 x - R = 576 x - 9 S = 9 (64 x - S) (S = block sum; W_00 = 576 / 64 = 9) and
    # sse576 = 81 sum (64 x - S)^2 — brute force over the blocks, no transform involved
    img = S.corpus_c2(2, 32, 48)
    want = []
    for im in img.astype(np.int64):
        tot = 0
        for by in range(0, 32, 8):
            for bx in range(0, 48, 8):
                b = im[by:by + 8, bx:bx + 8]
                tot += int(81 * ((64 * b - b.sum()) ** 2).sum())
        want.append(tot)
    assert O.compress_zonal_sse576(img, 1).tolist() == want
    assert np.all(O.compress_zonal_sse576(img, 64) == 0)          # P8: r = 64 is lossless
    assert O.compress_zonal_sse576(img, 10).dtype == np.int64


def test_P10_sse_monotone_in_r():
    img = S.corpus_c2(3, 64, 64)
    prev = None
    for r in range(1, 65):
        s = O.compress_zonal_sse(img, r)
        if prev is not None:
            assert np.all(s <= prev + 1e-7)
        prev = s
    assert np.all(prev < 1e-12)


def test_P15_impulse_responses_kronecker():
    T = O.c0_matrix()
    d = np.array([8, 6, 4, 6, 8, 6, 4, 6])
    W = 576 // np.outer(d, d)
    K = np.kron(T, T)                                       # vec_row(T X T^T) = (T (x) T) vec_row(X)
    for r in (1, 3, 10, 36, 64):
        G = K.T @ np.diag((W * O.zonal_mask(r)).ravel()) @ K   # 576 x_hat = G x
        for p in range(64):
            X = np.zeros((8, 8), dtype=np.uint8)
            X[p // 8, p % 8] = 1
            R = O.reconstruct_zonal_exact(X, r)[0]
            assert np.array_equal(R.ravel(), G[:, p])
            assert np.abs(O.reconstruct_zonal(X, r)[0].ravel() - G[:, p] / 576).max() < 1e-12


def test_P17_pattern_blocks_closed_form():
    T = O.c0_matrix()
    d = np.array([8, 6, 4, 6, 8, 6, 4, 6])
    img, I, J, A = S.pattern_image_from_rows(T, 64, 128, seed=5)
    Y = O.to_blocks(O.forward_int(img))[0]
    for by in range(I.shape[0]):
        for bx in range(I.shape[1]):
            i, j, a = I[by, bx], J[by, bx], A[by, bx]
            exp = np.zeros((8, 8), dtype=np.int64)
            exp[0, 0] += 8192
            exp[i, j] += a * d[i] * d[j]
            assert np.array_equal(Y[by, bx], exp)
    zz = O.zigzag_index()
    for r in (1, 3, 10, 36, 64):
        want = sum(0 if zz[I[b], J[b]] < r else A[b] ** 2 * d[I[b]] * d[J[b]] for b in np.ndindex(I.shape))
        got = O.compress_zonal_sse(img, r)[0]
        assert abs(got - want) <= 1e-8 * max(1, want)


# ---------------------------------------------------------------- quantiser (R10, P14, P18)

def test_quantize_exact_ties_round_away():
    d = np.array([8, 6, 4, 6, 8, 6, 4, 6])
    # put Y on an exact tie at (0,0): Z = Y/8, Z/q = Y/128 -> Y = 64 is 0.5 exactly
    for y, k in [(64, 1), (-64, -1), (63, 0), (-63, 0), (192, 2), (-192, -2), (65, 1)]:
        Y = np.zeros((8, 8), dtype=np.int64)
        Y[0, 0] = y
        assert O.quantize_exact(Y, 16.0)[0, 0, 0] == k
    # (2,2): dd = 16, Z/q = Y / 64; (1,1): dd = 36 -> Y / 96
    Y = np.zeros((8, 8), dtype=np.int64)
    Y[2, 2], Y[1, 1] = -32, 48
    k = O.quantize_exact(Y, 16.0)[0]
    assert k[2, 2] == -1 and k[1, 1] == 1
    # non-integer step uses exact rational arithmetic
    Y[0, 0] = 3
    assert O.quantize_exact(Y, 0.75)[0, 0, 0] == 1   # 3/8/0.75 = 0.5 -> 1


def test_P14_quantizer_exact_vs_decimal_brute_force():
    """k = round_half_away(Y / (q sqrt(d_i d_j))) recomputed with 60-digit decimal arithmetic."""
    from decimal import Decimal, ROUND_HALF_UP, getcontext
    getcontext().prec = 60
    d = [8, 6, 4, 6, 8, 6, 4, 6]
    Ys = np.arange(-1500, 1501)
    for q in (16.0, 0.75, 5.0):
        for (i, j) in [(0, 0), (1, 1), (0, 1), (2, 3), (2, 2), (7, 5)]:
            Y = np.zeros((len(Ys), 8, 8), dtype=np.int64)
            Y[:, i, j] = Ys
            img = O.from_blocks(Y[:, None, None])
            k = O.to_blocks(O.quantize_exact(img, q))[:, 0, 0, i, j]
            den = Decimal(q) * Decimal(d[i] * d[j]).sqrt()
            for y, kk in zip(Ys.tolist(), k.tolist()):
                want = int((Decimal(y) / den).quantize(Decimal(1), rounding=ROUND_HALF_UP))
                assert kk == want, (q, i, j, y, kk, want)


def _reachable_y_range(i, j):
    """[lo, hi] of Y_ij = sum_mn T_im T_jn x_mn over all uint8 blocks (every integer in between is
    reachable: the outer-product entries are in {0, +-1})."""
    T = golden_c0()
    P = np.outer(T[i], T[j])
    return int(255 * P[P < 0].sum()), int(255 * P[P > 0].sum())


@pytest.mark.parametrize("q", [16.0])
def test_P14_quantizer_full_reachable_domain(q):
    """P14 on the whole input domain: for every position (i, j) and every reachable Y_ij, the oracle's exact decision equals round_half_away(Y / (q sqrt(d_i d_j)))
    recomputed with 60-digit decimal arithmetic (Decimal ROUND_HALF_UP = ties away from zero).
    The domain is every reachable Y at every position (587,584 pairs)."""
    from decimal import Decimal, ROUND_HALF_UP, getcontext
    getcontext().prec = 60
    d = [8, 6, 4, 6, 8, 6, 4, 6]
    total = 0
    memo = {}
    for i in range(8):
        for j in range(8):
            lo, hi = _reachable_y_range(i, j)
            Ys = np.arange(lo, hi + 1)
            total += len(Ys)
            Y = np.zeros((len(Ys), 8, 8), dtype=np.int64)
            Y[:, i, j] = Ys
            k = O.to_blocks(O.quantize_exact(O.from_blocks(Y[:, None, None]), q))[:, 0, 0, i, j]
            dd = d[i] * d[j]
            if dd not in memo:
                den = Decimal(q) * Decimal(dd).sqrt()
                yall = np.arange(-16320, 16321)
                memo[dd] = dict(zip(yall.tolist(), [int((Decimal(y) / den).quantize(Decimal(1), rounding=ROUND_HALF_UP))
                                                    for y in yall.tolist()]))
            want = np.array([memo[dd][y] for y in Ys.tolist()])
            bad = np.nonzero(k != want)[0]
            assert len(bad) == 0, (i, j, Ys[bad[:5]], k[bad[:5]], want[bad[:5]])
    # 587,584 reachable (position, Y) pairs (SURVEY §8(c) quotes 620,224 for a looser per-position range;
    # every integer between the exact extremes of sum_mn T_im T_jn x_mn is reachable and is covered here)
    assert total == 587584


def test_quant_zonal_r_parseval_identity():
    """Reading R17 (quantiser with zonal r): by the orthogonality of C the pixel-domain SSE of
    C^T (q M_r k) C equals the coefficient-domain energy sum_kept (Z - q k)^2 + sum_discarded Z^2, an
    identity the oracle's literal inverse must satisfy for every r (a dropped mask, a wrong index or a
    transposed operand in the composition breaks it)."""
    imgs = np.concatenate([S.corpus_c2(3, 32, 48), rng.integers(0, 256, (2, 32, 48), dtype=np.uint8)])
    Zb = O.to_blocks(O.forward_scaled(imgs))
    for q in (16.0, 5.0, 350.0):
        kb = O.to_blocks(O.quantize_exact(O.forward_int(imgs), q)).astype(np.float64)
        for r in (1, 2, 10, 36, 63, 64):
            M = O.zonal_mask(r)
            want = (np.where(M, Zb - q * kb, Zb) ** 2).sum(axis=(1, 2, 3, 4))
            got = O.compress_quant_sse(imgs, q, r)
            assert np.allclose(got, want, rtol=1e-9, atol=1e-6), (q, r)
    assert np.array_equal(O.reconstruct_quant(imgs, 16.0, 64), O.reconstruct_quant(imgs, 16.0))


def test_quant_zonal_r_limits():
    """Tiny step: the quantised zonal reconstruction tends to the plain zonal one (each kept
    coefficient moves by at most q/2, so SSE differs by <= n_kept q^2 / 4 + 2 sqrt(SSE n_kept) q / 2);
    huge step (q > 2 max|Z|): every k = 0, x^ = 0, SSE = sum x^2 for every r."""
    imgs = S.corpus_c2(2, 32, 32)
    nblk = imgs.shape[0] * 16
    for r in (1, 6, 21, 50):
        q = 1.0 / 1024
        sz = O.compress_zonal_sse(imgs, r)
        sq = O.compress_quant_sse(imgs, q, r)
        nk = r * nblk / imgs.shape[0]
        assert np.all(np.abs(sq - sz) <= nk * q * q / 4 + q * np.sqrt(sz * nk) + 1e-9), r
        big = O.compress_quant_sse(imgs, 8192.0, r)
        assert np.allclose(big, (imgs.astype(np.float64) ** 2).sum(axis=(1, 2)), rtol=1e-12)


def test_P18_quant_constant_image_closed_form():
    for v in range(256):
        img = np.full((8, 16), v, dtype=np.uint8)
        rec = O.reconstruct_quant(img, 16.0)
        want = 2 * math.floor(v / 2 + 0.5)
        assert np.abs(rec - want).max() < 1e-9
        sse = O.compress_quant_sse(img, 16.0)[0]
        assert abs(sse - (0 if v % 2 == 0 else 128)) < 1e-7
        # a constant block has only the DC coefficient, which every r >= 1 keeps (R17)
        assert abs(O.compress_quant_sse(img, 16.0, 1)[0] - sse) < 1e-7


def test_inverse_from_coefficients_and_exact_u8_rounding():
    """reconstruct_from_coef_exact on a forward's output equals the pinned zonal twin (P8 / P15), its
    r = 64 inverse of any plane equals 576 x the float64 literal inverse C^T (D Y D) C, and
    round_u8_exact576 equals round_u8 of R / 576 away from exact ties and rounds ties away from 0."""
    imgs = np.concatenate([S.corpus_c2(2, 16, 24), rng.integers(0, 256, (2, 16, 24), dtype=np.uint8)])
    for r in (1, 10, 36, 64):
        assert np.array_equal(O.reconstruct_from_coef_exact(O.forward_int(imgs), r), O.reconstruct_zonal_exact(imgs, r))
    Y = rng.integers(-32768, 32768, (3, 16, 24))
    d = np.array([8, 6, 4, 6, 8, 6, 4, 6], dtype=float)
    Z = O.from_blocks(O.to_blocks(Y) / np.sqrt(np.outer(d, d)))
    R = O.reconstruct_from_coef_exact(Y, 64)
    assert np.allclose(R / 576.0, O.inverse(Z), rtol=1e-12, atol=1e-6)
    R = np.array([-1000, -289, -288, -1, 0, 287, 288, 289, 863, 864, 146591, 146592, 10 ** 7])
    assert O.round_u8_exact576(R).tolist() == [0, 0, 0, 0, 0, 0, 1, 1, 1, 2, 254, 255, 255]


def test_u8_rounding():
    x = np.array([-3.2, 0.49, 0.5, 254.5, 255.2, 300.0, 12.5, 13.5])
    assert O.round_u8(x).tolist() == [0, 0, 1, 255, 255, 255, 13, 14]


# ---------------------------------------------------------------- metrics, edge cases

def test_psnr_mean_and_edge_cases():
    assert O.mean_psnr([1.0 * 64, 4.0 * 64], 64) == pytest.approx(
        0.5 * (20 * math.log10(255) + 10 * math.log10(255 ** 2 / 4)))
    empty = np.zeros((0, 8, 8), dtype=np.uint8)
    assert O.forward_int(empty).shape == (0, 8, 8)
    assert O.compress_zonal_sse(empty, 10).shape == (0,)
    with pytest.raises(ValueError):
        O.to_blocks(np.zeros((12, 16), dtype=np.uint8))


def test_synth_generators_shapes_and_ranges():
    a = S.image_c1(0)
    assert a.shape == (512, 512) and a.dtype == np.uint8
    assert np.array_equal(a, S.image_c1(0))
    c = S.corpus_c2(6, 64, 64)
    assert c.shape == (6, 64, 64)
    assert len({c[i].tobytes() for i in range(6)}) == 6
    assert 20 < a.std() < 80


# ---------------------------------------------------------------- UQI / APE (F2, reading R16)

def brute_uqi(a, b, wdw=8):
    """Python-loop UQI with (N-1)-normalised moments, as in the Wang-Bovik definition."""
    h, w = a.shape
    tot, cnt = 0.0, 0
    for i in range(h - wdw + 1):
        for j in range(w - wdw + 1):
            xs = [float(v) for v in a[i:i + wdw, j:j + wdw].ravel()]
            ys = [float(v) for v in b[i:i + wdw, j:j + wdw].ravel()]
            N = len(xs)
            mx, my = sum(xs) / N, sum(ys) / N
            vx = sum((v - mx) ** 2 for v in xs) / (N - 1)
            vy = sum((v - my) ** 2 for v in ys) / (N - 1)
            c = sum((p - mx) * (q - my) for p, q in zip(xs, ys)) / (N - 1)
            d1, d2 = vx + vy, mx * mx + my * my
            lum = 1.0 if d2 <= 1e-12 else 2 * mx * my / d2
            ctr = 1.0 if d1 <= 1e-12 * (N / (N - 1)) else 2 * c / d1
            q_ = lum * ctr
            tot += q_
            cnt += 1
    return tot / cnt


def test_uqi_brute_force_and_properties():
    a = rng.integers(0, 256, size=(16, 16)).astype(float)
    b = np.clip(a + rng.normal(0, 20, size=a.shape), 0, 255)
    assert abs(O.uqi(a, b) - brute_uqi(a, b)) < 1e-12          # 1/N vs 1/(N-1) cancels
    assert abs(O.uqi(a, b) - O.uqi(b, a)) < 1e-15              # symmetric
    assert abs(O.uqi(3.5 * a, 3.5 * b) - O.uqi(a, b)) < 1e-12   # common-scale invariant
    assert abs(O.uqi(a, a) - 1.0) < 1e-12                      # identical non-constant -> 1
    inv = 255 - a
    assert O.uqi(a, inv) < 0                                   # anticorrelated windows
    c = np.full((12, 12), 7.0)
    assert O.uqi(c, c) == 1.0                                  # R16: both constant, equal
    assert abs(O.uqi(c, 2 * c) - 2 * 7 * 14 / (49 + 196)) < 1e-15
    z = np.zeros((9, 9))
    assert O.uqi(z, z) == 1.0
    osc = np.tile([[-5.0, 5.0], [5.0, -5.0]], (6, 6))          # zero mean, non-flat vs a black window
    assert O.uqi(np.zeros((12, 12)), osc) == 0.0
    assert abs(O.uqi(c, c + 1e-9 * rng.normal(size=c.shape)) - 1.0) < 1e-9   # round-off on a flat region
    with pytest.raises(ValueError):
        O.uqi(np.zeros((4, 4)), np.zeros((4, 4)))
    assert O.ape(1.1, 1.0) == pytest.approx(10.0)
    assert O.ape(2.0, 2.0) == 0.0
