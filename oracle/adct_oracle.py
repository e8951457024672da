"""CPU ORACLE for the arXiv 1402.6034 hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product path
(``paper_1402_6034_b200``) never imports it, and this module imports nothing
from the product path: the two share no code, headers, tables or constants.

Plain, slow, obviously-correct numpy, float64 unless an integer result is
exact.  Every step follows the plain definition from the paper; there is no
butterfly, blocking or fusion here (the fast algorithm of Fig. 1 is an exact
factorisation of C0, so the plain matrix product *is* the definition it
reaches).

Citations: ``P:n`` = /root/reference/PAPER.md line n (LaTeX source of the
paper); section names follow the paper.  Readings where the paper is silent
or garbled are numbered R1..R19 and listed in DESIGN.md §3.

Parity pins: every public function here is pinned by ``tests/test_oracle_pins.py``
against values the paper prints (``tests/golden/``), closed forms, invariants
or brute force.  ``transfer_error_energy`` is pinned by Table 2 only.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

__all__ = [
    "dct_matrix", "round_half_away", "c0_matrix", "orthogonalizer", "proposed_matrix",
    "coarse_matrix", "frobenius_optimal_scale", "sdct_matrix", "transfer_error_energy",
    "roundoff_matrix", "polar_orthogonal", "ceil_matrix", "sdct_sign_matrix",
    "zigzag_order", "zigzag_index", "zonal_mask", "to_blocks", "from_blocks",
    "forward_int", "forward_scaled", "inverse", "reconstruct_zonal", "reconstruct_zonal_exact",
    "reconstruct_from_coef_exact", "round_u8_exact576",
    "quantize_exact", "reconstruct_quant", "sse_per_image", "psnr", "mean_psnr",
    "compress_zonal_sse", "compress_zonal_sse576", "compress_quant_sse", "round_u8", "uqi", "ape",
]


# --------------------------------------------------------------------------------------
# §2 "DCT round-off approximations" — matrix construction
# --------------------------------------------------------------------------------------

def dct_matrix() -> np.ndarray:
    """Exact 8-point DCT matrix C ("the standard DCT matrix C").

    Reading R1: the paper does not print C; "standard" is taken as the orthonormal
    DCT-II, C[m][n] = a_m cos((2n+1) m pi / 16), a_0 = 1/(2 sqrt 2), a_m = 1/2.
    Pinned by Table 2 and the 0.3922 scale.
    """
    C = np.empty((8, 8), dtype=np.float64)
    for m in range(8):
        a = 1.0 / (2.0 * math.sqrt(2.0)) if m == 0 else 0.5
        for n in range(8):
            C[m, n] = a * math.cos((2 * n + 1) * m * math.pi / 16.0)
    return C


def round_half_away(x):
    """Round-off "[.]" as implemented in Matlab: nearest integer, ties away from 0."""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.floor(np.abs(x) + 0.5)


def c0_matrix() -> np.ndarray:
    """C0 = [2 C]: scale by two, then element-wise round-off. int64."""
    return round_half_away(2.0 * dct_matrix()).astype(np.int64)


def orthogonalizer(C0: np.ndarray | None = None) -> np.ndarray:
    """S = sqrt((C0 C0^T)^-1), principal square root.

    Computed as the general principal root of the SPD matrix (C0 C0^T)^-1 through its
    eigendecomposition — not by assuming the result is diagonal; the pins check that it
    comes out as the printed diag(1/(2 sqrt2), 1/sqrt6, 1/2, ...).
    """
    if C0 is None:
        C0 = c0_matrix()
    G = C0.astype(np.float64) @ C0.astype(np.float64).T
    Ginv = np.linalg.inv(G)
    w, V = np.linalg.eigh(Ginv)
    if np.any(w <= 0):
        raise ValueError("C0 C0^T is not positive definite")
    return (V * np.sqrt(w)) @ V.T


def proposed_matrix() -> np.ndarray:
    """C_orth = S . C0, the proposed orthogonal approximation."""
    C0 = c0_matrix()
    return orthogonalizer(C0) @ C0.astype(np.float64)


def coarse_matrix() -> np.ndarray:
    """Coarse non-orthogonal approximation C_hat = 1/2 C0."""
    return 0.5 * c0_matrix().astype(np.float64)


def roundoff_matrix(kind: str = "round", alpha: float = 2.0) -> np.ndarray:
    """The paper's constructive family f(alpha C) (P:131-151 with f = round-off, alpha = 2) and the
    generalisations the conclusion proposes, "usual floor and ceiling functions can be considered
    instead of the round-off function", SURVEY §8(f) F4.  int64."""
    f = {"round": round_half_away, "floor": np.floor, "ceil": np.ceil}[kind]
    return np.asarray(f(alpha * dct_matrix()), dtype=np.float64).astype(np.int64)


def polar_orthogonal(T: np.ndarray) -> np.ndarray:
    """S . T with S = sqrt((T T^T)^-1) (principal root): the orthogonal polar factor of
    an invertible T.  For T = C0 this is the proposed C_orth (S diagonal); for a general
    round-off variant S is a dense symmetric matrix (no fast algorithm, F4)."""
    T = np.asarray(T, dtype=np.float64)
    return orthogonalizer(T) @ T


def ceil_matrix() -> np.ndarray:
    """F4 variant: the orthogonal polar factor of ceil(2 C).  ceil(2 C) has entries
    in {0, 1} and is invertible (det 16); its Gram matrix is not diagonal, so S is dense."""
    return polar_orthogonal(roundoff_matrix("ceil"))


def sdct_sign_matrix() -> np.ndarray:
    """sign(C) (int64, entries +-1): the SDCT comparator is sign(C) / (2 sqrt 2) (R11)."""
    return np.sign(dct_matrix()).astype(np.int64)


def frobenius_optimal_scale() -> float:
    """argmin_a ||a C0 - C||_F = tr(C0^T C) / tr(C0^T C0) ("0.3922")."""
    C0 = c0_matrix().astype(np.float64)
    C = dct_matrix()
    return float(np.trace(C0.T @ C) / np.trace(C0.T @ C0))


def sdct_matrix() -> np.ndarray:
    """SDCT comparator: sign(C) scaled by 1/(2 sqrt2).

    Reading R11: the paper does not print the SDCT normalisation; 1/(2 sqrt 2) is the one
    that reproduces Table 2's SDCT column (pinned there). Not on the hot path.
    """
    return np.sign(dct_matrix()) / (2.0 * math.sqrt(2.0))


def transfer_error_energy(T: np.ndarray, n_grid: int = 20001) -> np.ndarray:
    """epsilon_m(T) = int_0^pi |H_m(w;C) - H_m(w;T)|^2 dw, m = 0..7.

    H_m(w;T) = sum_n t_{m,n} exp(-j n w); D_m = |H_m(C) - H_m(T)|^2;
    "numerically evaluated" — composite Simpson rule on n_grid points.
    """
    C = dct_matrix()
    w = np.linspace(0.0, math.pi, n_grid)
    E = np.exp(-1j * np.outer(np.arange(8), w))  # [n, w]
    Hc = C @ E
    Ht = np.asarray(T, dtype=np.float64) @ E
    D = np.abs(Hc - Ht) ** 2
    h = w[1] - w[0]
    wts = np.ones(n_grid)
    wts[1:-1:2] = 4.0
    wts[2:-1:2] = 2.0
    return (D * wts).sum(axis=1) * h / 3.0


# --------------------------------------------------------------------------------------
# §3 "Application to image compression" — zig-zag, blocks, 2-D transform
# --------------------------------------------------------------------------------------

def zigzag_order() -> list[tuple[int, int]]:
    """The standard zig-zag sequence (cited to [pao1998]); reading R4 = JPEG order.

    Generated by rule: anti-diagonals s = i + j ascending; on odd s the row index i
    ascends, on even s the column index j ascends (so index 1 is (0,1), index 2 is (1,0)).
    (i, j) = (row / vertical frequency, column / horizontal frequency).
    """
    order = []
    for s in range(15):
        cells = [(i, s - i) for i in range(8) if 0 <= s - i < 8]
        if s % 2 == 0:
            cells.sort(key=lambda c: c[1])   # j ascending
        else:
            cells.sort(key=lambda c: c[0])   # i ascending
        order.extend(cells)
    return order


def zigzag_index() -> np.ndarray:
    """8x8 int array: zig-zag position of coefficient (i, j)."""
    Z = np.empty((8, 8), dtype=np.int64)
    for k, (i, j) in enumerate(zigzag_order()):
        Z[i, j] = k
    return Z


def zonal_mask(r: int) -> np.ndarray:
    """M_r: keep "only the r initial coefficients" of the zig-zag sequence."""
    if not (1 <= r <= 64):
        raise ValueError("r must be in [1, 64]")
    return zigzag_index() < r


def to_blocks(img: np.ndarray) -> np.ndarray:
    """Partition [n, h, w] into non-overlapping 8x8 sub-blocks -> [n, h/8, w/8, 8, 8]."""
    img = np.asarray(img)
    if img.ndim == 2:
        img = img[None]
    n, h, w = img.shape
    if h % 8 or w % 8:
        raise ValueError("image dimensions must be multiples of 8 (reading R9)")
    return img.reshape(n, h // 8, 8, w // 8, 8).transpose(0, 1, 3, 2, 4)


def from_blocks(B: np.ndarray) -> np.ndarray:
    """Inverse of to_blocks: [n, H, W, 8, 8] -> [n, 8H, 8W] (coefficients in place, reading R12)."""
    n, H, W = B.shape[:3]
    return B.transpose(0, 1, 3, 2, 4).reshape(n, 8 * H, 8 * W)


def forward_int(img: np.ndarray) -> np.ndarray:
    """Y = T . A . T^T per block with T = C0, exact int64, image-shaped."""
    T = c0_matrix()
    B = to_blocks(img).astype(np.int64)
    return from_blocks(T @ B @ T.T)


def forward_scaled(img: np.ndarray, T: np.ndarray | None = None) -> np.ndarray:
    """Z = T . A . T^T per block in float64 with T = C_orth by default, image-shaped."""
    if T is None:
        T = proposed_matrix()
    B = to_blocks(img).astype(np.float64)
    return from_blocks(T @ B @ T.T)


def inverse(Z: np.ndarray, T: np.ndarray | None = None) -> np.ndarray:
    """Inverse procedure: A_hat = T^T . Z . T per block (T orthogonal)."""
    if T is None:
        T = proposed_matrix()
    B = to_blocks(Z).astype(np.float64)
    return from_blocks(T.T @ B @ T)


def _mask_image(Z: np.ndarray, r: int) -> np.ndarray:
    B = to_blocks(Z)
    return from_blocks(B * zonal_mask(r))


def reconstruct_zonal(img: np.ndarray, r: int, T: np.ndarray | None = None) -> np.ndarray:
    """Forward, keep the first r zig-zag coefficients, inverse. float64."""
    if T is None:
        T = proposed_matrix()
    Z = forward_scaled(img, T)
    return inverse(_mask_image(Z, r), T)


def reconstruct_zonal_exact(img: np.ndarray, r: int) -> np.ndarray:
    """Exact-integer twin of reconstruct_zonal for the proposed transform.

    With C = S C0 and S = diag(d)^-1/2, C^T (M . Z) C = C0^T (S (M . Y) S) C0 and
    S_ii S_jj = 1/sqrt(d_i d_j); 576 / (d_i d_j) is an integer W_ij for d = (8,6,4,6,...).
    Returns R = C0^T (W . M . Y) C0 (int64) with A_hat = R / 576 exactly.
    """
    T = c0_matrix()
    d = np.diag(T @ T.T)
    W = 576 // np.outer(d, d)
    assert np.all(W * np.outer(d, d) == 576)
    Y = to_blocks(forward_int(img))
    V = Y * (W * zonal_mask(r))
    return from_blocks(T.T @ V @ T)


def reconstruct_from_coef_exact(Y: np.ndarray, r: int) -> np.ndarray:
    """Exact-integer inverse of an arbitrary integer coefficient plane Y (image-shaped, R12):
    R = C0^T (W . M_r . Y) C0 per block (int64), so the reconstruction is R / 576 exactly — the
    inverse procedure with C^T and S folded into integer weights, the same
    composition as reconstruct_zonal_exact but from given coefficients instead of a forward."""
    T = c0_matrix()
    d = np.diag(T @ T.T)
    W = 576 // np.outer(d, d)
    V = to_blocks(np.asarray(Y)).astype(np.int64) * (W * zonal_mask(r))
    return from_blocks(T.T @ V @ T)


def round_u8_exact576(R: np.ndarray) -> np.ndarray:
    """clamp(round_half_away(R / 576), 0, 255) decided on the exact integer R (reading R3): for
    R >= 0, floor((R + 288) / 576); every negative R clamps to 0."""
    R = np.asarray(R, dtype=np.int64)
    return np.clip(np.floor_divide(R + 288, 576), 0, 255).astype(np.uint8)


def quantize_exact(Y: np.ndarray, q: float) -> np.ndarray:
    """k_ij = round_half_away(Z_ij / q) with Z_ij = Y_ij / sqrt(d_i d_j), decided EXACTLY.

    Reading R10 (BASELINE C4 "D-scaled uniform quantisation with step q"; the paper only says
    S is merged into the quantisation step): one step q for all 64 orthonormal
    coefficients, Matlab round.  |k| = max{k >= 0 : k = 0 or
    (2k-1)^2 q^2 d_i d_j <= 4 Y^2} — exact integer / rational arithmetic, so ties
    (|Z/q| = m + 1/2 exactly) always round away from zero.  Y is image-shaped int.
    """
    T = c0_matrix()
    d = np.diag(T @ T.T).astype(np.int64)
    Yb = to_blocks(np.asarray(Y)).astype(np.int64)
    dd = np.outer(d, d)
    qf = Fraction(q)
    if qf <= 0:
        raise ValueError("q must be > 0")
    num, den = qf.numerator, qf.denominator     # q = num / den exactly (float is dyadic)
    absY = np.abs(Yb)
    # float estimate, then exact correction with the integer predicate
    k = np.floor(absY / (float(q) * np.sqrt(dd)) + 0.5).astype(np.int64)
    kmax = int(k.max(initial=0)) + 2
    ymax = int(absY.max(initial=0))
    small = (2 * kmax + 1) ** 2 * num * num * 64 < 2 ** 62 and 4 * ymax * ymax * den * den < 2 ** 62
    dt = np.int64 if small else object          # Python ints when int64 could overflow
    lhs_scale = (num * num) * dd.astype(dt)      # (2k-1)^2 q^2 dd <= 4 Y^2  <=>  (2k-1)^2 num^2 dd <= 4 Y^2 den^2
    rhs = 4 * absY.astype(dt) * absY.astype(dt) * (den * den)

    def ok(kk):  # predicate "(2kk-1)^2 num^2 dd <= 4 Y^2 den^2" (True for kk <= 0)
        t = 2 * kk.astype(dt) - 1
        return np.where(kk <= 0, True, (t * t * lhs_scale) <= rhs)

    for _ in range(3):
        up = ok(k + 1)
        k = np.where(up, k + 1, k)
        down = ~ok(k)
        k = np.where(down, k - 1, k)
    assert np.all(ok(k)) and not np.any(ok(k + 1))
    return from_blocks(np.sign(Yb) * k)


def reconstruct_quant(img: np.ndarray, q: float, r: int = 64) -> np.ndarray:
    """Forward, D-scaled uniform quantiser (step q), dequantise Z_hat = q k, inverse C^T (R10). float64.

    With r < 64 the zonal step is applied too: only the first r zig-zag coefficients are kept
     and quantised, the others are discarded (k = 0) — S merged into the quantisation
    step of the kept coefficients, reading R17."""
    C = proposed_matrix()
    k = quantize_exact(forward_int(img), q)
    if r < 64:
        k = _mask_image(k, r)
    return inverse(q * k.astype(np.float64), C)


def round_u8(x: np.ndarray) -> np.ndarray:
    """Optional 8-bit reconstruction: clamp(round_half_away(x), 0, 255) (reading R3, secondary)."""
    return np.clip(round_half_away(x), 0, 255).astype(np.uint8)


# --------------------------------------------------------------------------------------
# Figures of merit
# --------------------------------------------------------------------------------------

def sse_per_image(img: np.ndarray, rec: np.ndarray) -> np.ndarray:
    """Per-image sum of squared pixel differences (MSE = SSE / (h w)). float64."""
    a = np.asarray(img, dtype=np.float64)
    b = np.asarray(rec, dtype=np.float64)
    if a.ndim == 2:
        a, b = a[None], b[None]
    return ((a - b) ** 2).reshape(a.shape[0], a.shape[1] * a.shape[2]).sum(axis=1)


def psnr(sse, pixels: int, peak: float = 255.0):
    """PSNR = 10 log10(peak^2 / MSE), MSE = SSE / pixels; +inf for SSE = 0 (R7, R8)."""
    sse = np.asarray(sse, dtype=np.float64)
    with np.errstate(divide="ignore"):
        return np.where(sse == 0, np.inf, 10.0 * np.log10(peak * peak * pixels / np.where(sse == 0, 1, sse)))


def mean_psnr(sse, pixels: int) -> float:
    """"average PSNR from all images": arithmetic mean of per-image PSNR (R6)."""
    return float(np.mean(psnr(sse, pixels)))


def compress_zonal_sse(img: np.ndarray, r: int, T: np.ndarray | None = None) -> np.ndarray:
    """Per-image SSE of the zonal pipeline (fwd, keep r, inverse) on the unrounded reconstruction (R3)."""
    img = np.asarray(img)
    if img.ndim == 2:
        img = img[None]
    return sse_per_image(img, reconstruct_zonal(img, r, T))


def compress_zonal_sse576(img: np.ndarray, r: int) -> np.ndarray:
    """Exact integer twin of compress_zonal_sse: per-image sum of (576 x - R)^2 (int64), where
    576 A_hat = R = C0^T (W . M_r . Y) C0 (reconstruct_zonal_exact), so
    SSE = sse576 / 576^2 exactly (P:496-497 on the unrounded reconstruction, R3)."""
    img = np.asarray(img)
    if img.ndim == 2:
        img = img[None]
    e = 576 * img.astype(np.int64) - reconstruct_zonal_exact(img, r)
    return (e * e).reshape(img.shape[0], -1).sum(axis=1)


def compress_quant_sse(img: np.ndarray, q: float, r: int = 64) -> np.ndarray:
    """Per-image SSE of the quantiser pipeline (R10; zonal r as in reconstruct_quant, R17) on the
    unrounded reconstruction (R3)."""
    img = np.asarray(img)
    if img.ndim == 2:
        img = img[None]
    return sse_per_image(img, reconstruct_quant(img, q, r))


# --------------------------------------------------------------------------------------
# Universal quality index and APE (second workload)
# --------------------------------------------------------------------------------------

def uqi(a: np.ndarray, b: np.ndarray, window: int = 8) -> float:
    """Mean over all window x window sliding windows (stride 1) of the Wang-Bovik index
    Q = 4 s_xy mx my / ((s_x^2 + s_y^2)(mx^2 + my^2))  (sample moments; the 1/N vs 1/(N-1)
    normalisation cancels), i.e. Q = L * S with L = 2 mx my / (mx^2 + my^2) (luminance) and
    S = 2 s_xy / (s_x^2 + s_y^2) (correlation x contrast).  Reading R16 for degenerate windows:
    a 0/0 factor is 1 — L = 1 when mx^2 + my^2 <= 1e-12, S = 1 when s_x^2 + s_y^2 <= 1e-12
    (pixel^2 units; a non-flat or non-black 8-bit window is far above these: s_x^2 >= 63/64^2,
    mx^2 >= 1/64^2, so the guards only absorb floating-point round-off of the reconstruction).
    float64, moments about the window mean."""
    x = np.asarray(a, dtype=np.float64)
    y = np.asarray(b, dtype=np.float64)
    if x.shape != y.shape or x.ndim != 2:
        raise ValueError("uqi: two images of equal 2-D shape")
    if x.shape[0] < window or x.shape[1] < window:
        raise ValueError("uqi: image smaller than the window")
    from numpy.lib.stride_tricks import sliding_window_view as swv
    X = swv(x, (window, window))
    Y = swv(y, (window, window))
    mx = X.mean(axis=(2, 3))
    my = Y.mean(axis=(2, 3))
    dx = X - mx[..., None, None]
    dy = Y - my[..., None, None]
    vx = (dx * dx).mean(axis=(2, 3))
    vy = (dy * dy).mean(axis=(2, 3))
    cxy = (dx * dy).mean(axis=(2, 3))
    d1 = vx + vy
    d2 = mx * mx + my * my
    L = np.where(d2 <= 1e-12, 1.0, 2 * mx * my / np.where(d2 <= 1e-12, 1.0, d2))
    S_ = np.where(d1 <= 1e-12, 1.0, 2 * cxy / np.where(d1 <= 1e-12, 1.0, d1))
    return float((L * S_).mean())


def ape(value: float, reference: float) -> float:
    """Absolute percentage error relative to the exact-DCT value: 100 |v - ref| / |ref|."""
    if reference == 0:
        raise ValueError("ape: zero reference")
    return 100.0 * abs(value - reference) / abs(reference)
