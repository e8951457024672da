"""GPU parity for every mode the C ABI exposes beyond the headline path (round-2 additions):
the quantiser combined with a zonal r < 64, the inverse from int32 / f32 coefficient planes to u8,
saturating u8 reconstructions (coefficient planes and quantiser steps that drive x^ far outside
[0, 255]) and the per-lane u8 store path (w % 16 != 0).  Bars as tests/test_gpu_parity.py: integer
decisions exact, f32 within 1e-4 on the 0-255 scale, SSE within rtol 1e-5 (PSNR within 1e-3 dB).

u8 from an fp32 reconstruction (quantiser, f32 coefficient plane): the kernel rounds its fp32 x^, the
oracle its float64 x^; they agree except where x^ lies within the fp32 reconstruction error of a
rounding boundary k + 1/2, and there by one step (the same rule as the round-1 quantiser u8 test).
"""
import numpy as np
import pytest

import oracle as O
from synth import images as S

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_1402_6034_b200 as A  # noqa: E402
from test_gpu_parity import FP_TOL, check_sse, host  # noqa: E402

rng = np.random.default_rng(2024)


def dev(x):
    return A.to_device(x)


def assert_u8_near_ties(got, want_f, tol=1e-4):
    """u8 of an fp32 x^ vs round_u8 of the float64 x^: equal except within `tol` of a tie, by <= 1."""
    want = O.round_u8(want_f)
    diff = np.abs(got.astype(np.int64) - want.astype(np.int64))
    near = np.abs(np.abs(want_f - np.floor(want_f)) - 0.5) < tol
    assert diff.max() <= 1, int(diff.max())
    assert np.all(near[diff > 0]), int((diff > 0).sum())


# ------------------------------------------------------------------ quantiser with zonal r < 64 (R17)

@pytest.mark.parametrize("r", [1, 10, 36, 63])
@pytest.mark.parametrize("q", [16.0, 5.0])
def test_compress_quant_zonal_r_vs_oracle(r, q):
    """k = round_half_away(Z / q) on the first r zig-zag positions, 0 elsewhere (P:234-248, P:488-491,
    reading R17): SSE-only, f32 and u8 reconstructions against the oracle, both u8 store paths."""
    for w in (96, 264):
        imgs = np.concatenate([S.corpus_c2(3, 64, w), rng.integers(0, 256, (2, 64, w), dtype=np.uint8)])
        want = O.reconstruct_quant(imgs, q, r)
        x = dev(imgs)
        sse = host(A.compress_psnr(x, r, q=q))
        check_sse(sse, O.sse_per_image(imgs, want), 64 * w)
        sse_f, rec = A.compress_psnr(x, r, q=q, recon="f32")
        assert np.abs(host(rec) - want).max() <= FP_TOL
        check_sse(host(sse_f), O.sse_per_image(imgs, want), 64 * w)
        _, rec8 = A.compress_psnr(x, r, q=q, recon="u8")
        assert_u8_near_ties(host(rec8), want)


def test_compress_quant_zonal_r_c4_frame():
    """C4 frame size (4320 x 7680), q = 16 with r = 10 and r = 36: SSE vs the oracle."""
    x = S.device_video(1, 4320, 7680, seed=0, first_frame=30)
    imgs = host(x)
    for r in (10, 36):
        check_sse(host(A.compress_psnr(x, r, q=16.0)), O.compress_quant_sse(imgs, 16.0, r), 4320 * 7680)


# ------------------------------------------------------------------ saturating u8 reconstructions

# A 0/255 block whose quantiser reconstruction at q = 400 reaches -457 (found by a greedy pixel-flip
# search over 120 random 0/255 starts minimising min(x^) with the float64 oracle, q in {300, 350, 400};
# an input fixture, not an expected value).
ADV_BLOCK = 255 * np.array([[1, 1, 0, 0, 1, 0, 0, 0], [1, 1, 0, 0, 1, 0, 1, 0], [1, 1, 1, 1, 0, 1, 1, 0],
                            [0, 1, 1, 0, 0, 0, 1, 1], [1, 1, 0, 1, 1, 1, 0, 1], [0, 1, 1, 1, 0, 0, 1, 1],
                            [1, 1, 1, 1, 1, 1, 1, 0], [1, 1, 1, 0, 0, 0, 1, 1]], dtype=np.uint8)


def test_quant_u8_clamps_far_below_zero():
    """The quantiser's u8 reconstruction saturates (x^ down to -457 here; the kernel's u8 rounding
    now clamps every input) on both u8 store paths."""
    q = 400.0
    assert O.reconstruct_quant(ADV_BLOCK, q).min() < -400
    imgs = np.concatenate([np.tile(ADV_BLOCK, (2, 4, 4)), np.tile(ADV_BLOCK.T, (1, 4, 4))])   # w % 16 == 0
    want = O.reconstruct_quant(imgs, q)
    _, rec8 = A.compress_psnr(dev(imgs), 64, q=q, recon="u8")
    assert_u8_near_ties(host(rec8), want)
    imgs2 = np.tile(ADV_BLOCK, (2, 2, 3))                 # 16 x 24: w % 16 != 0 (per-lane store path)
    _, rec8 = A.compress_psnr(dev(imgs2), 64, q=q, recon="u8")
    assert_u8_near_ties(host(rec8), O.reconstruct_quant(imgs2, q))


@pytest.mark.parametrize("coef", ["i16", "i32"])
@pytest.mark.parametrize("h,w", [(64, 96), (40, 272), (24, 264)])
def test_inverse_u8_saturating_integer_planes(coef, h, w):
    """Arbitrary integer coefficient planes (the full int16 range: x^ reaches far outside [0, 255]):
    u8 = clamp(round_half_away(R / 576)) on the exact integer R = C0^T (W . M . Y) C0 (oracle)."""
    Y = rng.integers(-32768, 32768, (3, h, w))
    Y[1] //= 64                                           # a milder plane: every node below 2^24, exact
    for r in (1, 10, 64):
        R = O.reconstruct_from_coef_exact(Y, r)
        got = host(A.inverse(dev(Y.astype(np.int16 if coef == "i16" else np.int32)), r=r, out="u8"))
        want = O.round_u8_exact576(R)
        assert np.array_equal(got[1], want[1]), r
        # full-range planes: fp32 inverse nodes exceed 2^24, so R is rounded by a few units; the
        # decision can then differ by one step only next to a rounding boundary (R = 576 k + 288)
        diff = np.abs(got.astype(np.int64) - want.astype(np.int64))
        m = (R + 288) % 576
        assert diff.max() <= 1 and np.all(np.minimum(m, 576 - m)[diff > 0] < 64), r
        assert np.mean(want == 0) > 0.1 and np.mean(want == 255) > 0.1    # saturation exercised


def test_inverse_i32_plane_beyond_2_22():
    """int32 coefficients with |Y| >= 2^22 convert exactly (I2FP) — the reconstruction
    matches the float64 oracle within its fp32 rounding (relative 1e-6 of the magnitude)."""
    Y = rng.integers(-2 ** 26, 2 ** 26, (2, 32, 64)).astype(np.int32)
    d = np.array([8, 6, 4, 6, 8, 6, 4, 6], dtype=float)
    Z = O.from_blocks(O.to_blocks(Y.astype(np.float64)) / np.sqrt(np.outer(d, d)))
    want = O.inverse(Z)
    got = host(A.inverse(dev(Y), r=64, out="f32"))
    assert np.abs(got - want).max() <= 1e-6 * np.abs(want).max()


# ------------------------------------------------------------------ inverse from i32 / f32 planes to u8

@pytest.mark.parametrize("h,w", [(64, 96), (40, 272), (24, 264)])
@pytest.mark.parametrize("r", [1, 10, 28, 64])
def test_inverse_u8_from_i32_and_f32_planes(h, w, r):
    """adct_inverse from the int32 Y plane (exact: u8 decided on the integer R) and from the f32 Z plane
    (near-tie rule) to u8, on the TMA bulk-store path (w % 16 == 0) and the per-lane path (w = 264)."""
    imgs = np.concatenate([S.corpus_c2(2, h, w), rng.integers(0, 256, (1, h, w), dtype=np.uint8)])
    Y = O.forward_int(imgs)
    got32 = host(A.inverse(dev(Y.astype(np.int32)), r=r, out="u8"))
    assert np.array_equal(got32, O.round_u8_exact576(O.reconstruct_zonal_exact(imgs, r)))
    Z = O.forward_scaled(imgs).astype(np.float32)
    gotf = host(A.inverse(dev(Z), r=r, out="u8"))
    assert_u8_near_ties(gotf, O.reconstruct_zonal(imgs, r))


def test_inverse_f32_plane_masked_nan_does_not_spread():
    """a NaN / Inf stored at a position the zonal mask discards must not reach the block."""
    imgs = S.corpus_c2(2, 32, 64)
    Z = O.forward_scaled(imgs).astype(np.float32)
    Zb = O.to_blocks(Z)
    zz = O.zigzag_index()
    Zb[..., zz >= 10] = np.nan
    Zb[..., 7, 7] = np.inf
    Zp = np.ascontiguousarray(O.from_blocks(Zb))
    rec = host(A.inverse(dev(Zp), r=10, out="f32"))
    assert np.all(np.isfinite(rec))
    assert np.abs(rec - O.reconstruct_zonal(imgs, 10)).max() <= FP_TOL
    # the per-lane path too (u8 planes with w % 16 != 0)
    imgs2 = S.corpus_c2(1, 16, 264)
    Zb2 = O.to_blocks(O.forward_scaled(imgs2).astype(np.float32))
    Zb2[..., zz >= 10] = np.nan
    rec8 = host(A.inverse(dev(np.ascontiguousarray(O.from_blocks(Zb2))), r=10, out="u8"))
    assert_u8_near_ties(rec8, O.reconstruct_zonal(imgs2, 10))


# ------------------------------------------------------------------ zonal u8 reconstruction, per-lane path

@pytest.mark.parametrize("w", [264, 520])
@pytest.mark.parametrize("r", [1, 10, 21, 36, 63])
def test_compress_zonal_u8_per_lane_store(w, r):
    """compress_psnr(recon='u8') with w % 16 != 0 (the per-lane store path): exact against the integer R."""
    imgs = np.concatenate([S.corpus_c2(2, 40, w), rng.choice(np.array([0, 255], np.uint8), size=(1, 40, w))])
    sse, rec8 = A.compress_psnr(dev(imgs), r, recon="u8")
    assert np.array_equal(host(rec8), O.round_u8_exact576(O.reconstruct_zonal_exact(imgs, r)))
    check_sse(host(sse), O.compress_zonal_sse(imgs, r), 40 * w)


# ------------------------------------------------------------------ canaries for the 32-bit inverse inputs

def _window(n, h, w, dtype, fill, pad_rows=8, pad_cols=32):
    es = torch.empty((), dtype=dtype).element_size()
    wp = -(-(w + pad_cols) * es // 16) * 16 // es
    big = torch.full((n + 1, h + pad_rows, wp), fill, dtype=dtype, device="cuda")
    return big, big[:n, :h, :w]


def _outside(big, n, h, w):
    m = torch.ones_like(big, dtype=torch.bool)
    m[:n, :h, :w] = False
    return big[m]


@pytest.mark.parametrize("n,h,w", [(3, 40, 264), (3, 40, 272), (1, 8, 8), (2, 24, 520)])
@pytest.mark.parametrize("coef", ["i16", "i32", "f32"])
def test_inverse_no_writes_outside_every_input_kind(n, h, w, coef):
    x = dev(rng.integers(0, 256, (n, h, w), dtype=np.uint8))
    y = A.forward(x, coef=coef)
    for out, dt, fill in [("f32", torch.float32, -12345.5), ("u8", torch.uint8, 77)]:
        for r in (10, 64):
            big, win = _window(n, h, w, dt, fill)
            A.inverse(y, r=r, out=out, dst=win)
            assert torch.all(_outside(big, n, h, w) == fill), (coef, out, r)
    torch.cuda.synchronize()


# ------------------------------------------------------------------ F1 SDCT fast path, F4 ceil variant

def _comparator_images(h=64, w=96):
    ii, jj = np.indices((h, w))
    return np.concatenate([S.corpus_c2(3, h, w), rng.integers(0, 256, (2, h, w), dtype=np.uint8),
                           (255 * ((ii + jj) % 2)).astype(np.uint8)[None], np.full((1, h, w), 255, np.uint8)])


@pytest.mark.parametrize("r", [1, 2, 3, 5, 10, 21, 36, 50, 63, 64])
def test_sdct_integer_fast_path_vs_oracle(r):
    """adct_compress_psnr_sdct (24-add SWAR forward, transposed 24-add inverse, e = 64 x - R exact)
    against the oracle's float64 pipeline with sign(C) / (2 sqrt 2) (R11): SSE within 1e-5."""
    for h, w in ((64, 96), (40, 264)):
        imgs = _comparator_images(h, w)
        got = host(A.compress_psnr_sdct(dev(imgs), r))
        want = O.compress_zonal_sse(imgs, r, O.sdct_matrix())
        check_sse(got, want, h * w)


def test_sdct_fast_path_matches_dense_and_c2_curve():
    """C2 (45 x 512^2): the SDCT mean-PSNR curve from the integer fast path equals the oracle's, and
    the fast path equals the dense fp32 comparator within the dense path's 1e-4."""
    imgs = S.corpus_c2()
    x = dev(imgs)
    px = 512 * 512
    for r in (1, 3, 6, 10, 15, 21, 28, 36, 45, 63):
        fast = host(A.compress_psnr_sdct(x, r))
        want = O.compress_zonal_sse(imgs, r, O.sdct_matrix())
        check_sse(fast, want, px)
        assert abs(O.mean_psnr(fast, px) - O.mean_psnr(want, px)) <= 1e-3
        assert np.allclose(fast, host(A.compress_psnr_dense(x, r, "sdct")), rtol=1e-4)


@pytest.mark.parametrize("r", [1, 3, 10, 21, 36, 50])
def test_dense_ceil_variant_vs_oracle(r):
    """F4: the polar factor of ceil(2C) (library's own Jacobi eigendecomposition) through the dense path
    vs the oracle's float64 pipeline with O.ceil_matrix(); fp32 dense products: SSE rtol 1e-4."""
    imgs = _comparator_images()
    got = host(A.compress_psnr_dense(dev(imgs), r, "ceil"))
    want = O.compress_zonal_sse(imgs, r, O.ceil_matrix())
    check_sse(got, want, 64 * 96, rtol=1e-4)
