"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle on the same seeded
inputs.  Bars (BASELINE.json north_star): integer coefficients bit-exact; fp32 coefficients and
reconstructions max |err| <= 1e-4 on the 0-255 scale; PSNR within 1e-3 dB.

SSE tolerance: each lane sums its 128 exact squared errors (576 x - 576 x^)^2
with fused fp32 FMAs, so the relative error of a lane's partial is at most 127 u = 7.6e-6
(u = 2^-24); partials are then combined in fp64.  SSE_RTOL = 1e-5 bounds that, and maps to
|dPSNR| <= 4.4e-5 dB, inside the 1e-3 dB bar.
"""
import math

import numpy as np
import pytest

import oracle as O
from synth import images as S

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_1402_6034_b200 as A  # noqa: E402

FP_TOL = 1e-4
SSE_RTOL = 1e-5
PSNR_TOL = 1e-3
rng = np.random.default_rng(99)


def dev(x):
    """16-byte-pitched device copy (the ABI requires pitch % 16 == 0)."""
    return A.to_device(x)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def check_sse(got, want, pixels, rtol=None):
    """SSE within SSE_RTOL (floor: MSE 1e-6) and PSNR within PSNR_TOL where the MSE is >= 1e-6.

    Below MSE 1e-6 (PSNR > 108 dB) both sides are lossless up to the oracle's own float64
    round-off (it reports ~1e-25 where the exact SSE is 0), so only the SSE bound applies.
    """
    got, want = np.asarray(got, float), np.asarray(want, float)
    floor = 1e-6 * pixels
    rtol = SSE_RTOL if rtol is None else rtol
    assert np.all(np.abs(got - want) <= rtol * np.maximum(np.abs(want), floor)), (got, want)
    big = want >= floor
    assert np.all(np.abs(O.psnr(got[big], pixels) - O.psnr(want[big], pixels)) <= PSNR_TOL)


def impulse_images():
    """128 single-block images: value 1 and value 255 at each of the 64 positions."""
    imgs = np.zeros((128, 8, 8), dtype=np.uint8)
    for p in range(64):
        imgs[p, p // 8, p % 8] = 1
        imgs[64 + p, p // 8, p % 8] = 255
    return imgs


def extreme_images():
    imgs = [np.zeros((8, 8)), np.full((8, 8), 255)]
    ii, jj = np.indices((8, 8))
    imgs += [255 * ((ii + jj) % 2), 255 * ((ii + jj + 1) % 2), 255 * (ii % 2), 255 * (jj % 2)]
    imgs += [rng.choice([0, 255], size=(8, 8)) for _ in range(58)]
    return np.stack(imgs).astype(np.uint8)


# ------------------------------------------------------------------ forward (integer, exact)

@pytest.mark.parametrize("coef", ["i16", "i32"])
def test_forward_integer_bit_exact_blocks(coef):
    for imgs in (impulse_images(), extreme_images(), rng.integers(0, 256, (300, 8, 8), dtype=np.uint8)):
        Y = host(A.forward(dev(imgs), coef=coef))
        assert np.array_equal(Y.astype(np.int64), O.forward_int(imgs))


@pytest.mark.parametrize("h,w", [(8, 8), (16, 16), (8, 504), (24, 520), (512, 512), (40, 264), (264, 8)])
def test_forward_shapes_and_ragged_tiles(h, w):
    imgs = rng.integers(0, 256, (3, h, w), dtype=np.uint8)
    Y = host(A.forward(dev(imgs)))
    assert np.array_equal(Y.astype(np.int64), O.forward_int(imgs))


def test_forward_c1_and_c3_subset_bit_exact():
    c1 = S.image_c1(0)
    assert np.array_equal(host(A.forward(dev(c1)))[0].astype(np.int64), O.forward_int(c1)[0])
    x = S.device_uniform(64, 512, 512, seed=0)       # C3 recipe, 64-image subset
    Y = host(A.forward(x)).astype(np.int64)
    assert np.array_equal(Y, O.forward_int(host(x)))


def test_forward_c3_full_size_bench_launch_sampled():
    """C3 in the launch configuration bench.py times: 8192 x 512^2 uniform images (2 GiB) -> int16
    (4 GiB) in ONE call; sampled images across the batch bit-exact against the oracle."""
    x = S.device_uniform(8192, 512, 512, seed=0)
    out = torch.empty((8192, 512, 512), dtype=torch.int16, device="cuda")
    A.forward(x, out=out)
    sample = [0, 1, 4095, 4096, 8190, 8191]
    Y = host(out[sample]).astype(np.int64)
    imgs = host(x[sample])
    del x, out
    torch.cuda.empty_cache()
    assert np.array_equal(Y, O.forward_int(imgs))


def test_forward_pitch_and_image_stride():
    base = torch.zeros((3, 40, 96), dtype=torch.uint8, device="cuda")
    imgs = rng.integers(0, 256, (3, 32, 64), dtype=np.uint8)
    base[:, :32, :64] = dev(imgs)
    view = base[:, :32, :64]                                   # pitch 96, image stride 40*96
    out = torch.full((3, 48, 80), 7, dtype=torch.int16, device="cuda")
    A.forward(view, out=out[:, :32, :64])
    got = host(out)
    assert np.array_equal(got[:, :32, :64].astype(np.int64), O.forward_int(imgs))
    assert np.all(got[:, 32:, :] == 7) and np.all(got[:, :, 64:] == 7)   # nothing written outside


@pytest.mark.parametrize("r", [1, 3, 5, 10, 21, 36, 50, 63])
def test_forward_masked(r):
    imgs = rng.integers(0, 256, (4, 32, 48), dtype=np.uint8)
    want = O.from_blocks(O.to_blocks(O.forward_int(imgs)) * O.zonal_mask(r))
    for coef in ("i16", "i32"):
        assert np.array_equal(host(A.forward(dev(imgs), r=r, coef=coef)).astype(np.int64), want)
    Z = host(A.forward(dev(imgs), r=r, coef="f32"))
    Zw = O.from_blocks(O.to_blocks(O.forward_scaled(imgs)) * O.zonal_mask(r))
    assert np.abs(Z - Zw).max() <= FP_TOL


def test_forward_scaled_f32():
    imgs = np.concatenate([extreme_images(), rng.integers(0, 256, (200, 8, 8), dtype=np.uint8)])
    Z = host(A.forward(dev(imgs), coef="f32"))
    assert np.abs(Z - O.forward_scaled(imgs)).max() <= FP_TOL


# ------------------------------------------------------------------ inverse

@pytest.mark.parametrize("r", [1, 4, 10, 28, 64])
def test_inverse_from_integer_and_scaled(r):
    imgs = np.concatenate([S.corpus_c2(3, 64, 64).reshape(-1, 64, 64)])
    want = O.reconstruct_zonal(imgs, r)
    Y = O.forward_int(imgs).astype(np.int16)
    rec = host(A.inverse(dev(Y), r=r, out="f32"))
    assert np.abs(rec - want).max() <= FP_TOL
    rec32 = host(A.inverse(dev(Y.astype(np.int32)), r=r))
    assert np.abs(rec32 - want).max() <= FP_TOL
    Z = O.forward_scaled(imgs).astype(np.float32)
    recz = host(A.inverse(dev(Z), r=r))
    assert np.abs(recz - want).max() <= FP_TOL
    u8 = host(A.inverse(dev(Y), r=r, out="u8"))
    R = O.reconstruct_zonal_exact(imgs, r)
    assert np.array_equal(u8, O.round_u8(R / 576.0))


# ------------------------------------------------------------------ fused compress (zonal)

def test_compress_c1_r10():
    """BASELINE C1: one 512x512 image, r = 10, PSNR."""
    img = S.image_c1(0)
    sse = host(A.compress_psnr(dev(img), 10))
    check_sse(sse, O.compress_zonal_sse(img, 10), 512 * 512)


def test_compress_every_r_c2_like():
    imgs = S.corpus_c2(6, 128, 128)
    x = dev(imgs)
    for r in range(1, 65):
        sse = host(A.compress_psnr(x, r))
        want = O.compress_zonal_sse(imgs, r)
        if r == 64:
            assert np.all(sse < 1e-6)
            assert np.all(np.isinf(host(A.psnr(A.compress_psnr(x, r), 128 * 128))))
        else:
            check_sse(sse, want, 128 * 128)


def test_compress_c2_full_mean_psnr():
    """BASELINE C2 (45 x 512^2): mean PSNR per r = 1..64 for the proposed transform vs the oracle."""
    imgs = S.corpus_c2()
    x = dev(imgs)
    for r in range(1, 64):
        sse = host(A.compress_psnr(x, r))
        want = O.compress_zonal_sse(imgs, r)
        check_sse(sse, want, 512 * 512)
        assert abs(O.mean_psnr(sse, 512 * 512) - O.mean_psnr(want, 512 * 512)) <= PSNR_TOL


@pytest.mark.parametrize("h,w", [(64, 96), (40, 264), (24, 520)])
def test_compress_sse576_bit_exact(h, w):
    """adct_compress_sse576: sum (576 x - R)^2 per image, bit-exact against the oracle's int64,
    every r, ragged tiles, plus the extreme images (all 0 / all 255 / checkerboards)."""
    imgs = np.concatenate([rng.integers(0, 256, (3, h, w), dtype=np.uint8),
                           S.corpus_c2(2, h, w),
                           np.zeros((1, h, w), np.uint8), np.full((1, h, w), 255, np.uint8),
                           (255 * ((np.arange(h)[:, None] + np.arange(w)[None]) % 2)).astype(np.uint8)[None]])
    x = dev(imgs)
    for r in range(1, 65):
        got = host(A.compress_sse576(x, r))
        assert np.array_equal(got, O.compress_zonal_sse576(imgs, r)), r
        if r in (1, 10, 36):  # and the fp32-accumulated fused path agrees within its stated bound
            check_sse(host(A.compress_psnr(x, r)), got / 576.0 ** 2, h * w)


def test_compress_sse576_c1_and_f64_output():
    img = S.image_c1(0)
    x = dev(img)
    sse = torch.empty(1, dtype=torch.float64, device="cuda")
    got = host(A.compress_sse576(x, 10, sse=sse))
    want = O.compress_zonal_sse576(img, 10)
    assert np.array_equal(got, want)
    assert host(sse)[0] == float(want[0]) / 331776.0


@pytest.mark.parametrize("r", [1, 3, 6, 10, 15, 21, 28, 36, 7, 50])
def test_compress_recon_f32_and_u8(r):
    imgs = np.concatenate([S.corpus_c2(3, 64, 96),
                           rng.choice(np.array([0, 255], dtype=np.uint8), size=(2, 64, 96))])
    want = O.reconstruct_zonal(imgs, r)
    sse, rec = A.compress_psnr(dev(imgs), r, recon="f32")
    assert np.abs(host(rec) - want).max() <= FP_TOL
    check_sse(host(sse), O.compress_zonal_sse(imgs, r), 64 * 96)
    sse2, rec8 = A.compress_psnr(dev(imgs), r, recon="u8")
    R = O.reconstruct_zonal_exact(imgs, r)
    assert np.array_equal(host(rec8), O.round_u8(R / 576.0))
    assert np.allclose(host(sse2), host(sse), rtol=1e-12)


@pytest.mark.parametrize("h,w", [(8, 8), (8, 16), (24, 504), (40, 264), (264, 8), (16, 520),
                                 (8, 131080), (65544, 8)])
def test_compress_ragged_shapes(h, w):
    """Ragged geometries through one r of every kernel form and inverse flavour (sinv_mode): scalar
    direct (1, 10), f32x2 direct (3), grouped f32x2 (11), hybrid (13), per-block loop (15, 21),
    residual with an injected column (23, 28), residual (36), lossless (64)."""
    imgs = rng.integers(0, 256, (5, h, w), dtype=np.uint8)
    for r in (1, 3, 10, 11, 13, 15, 21, 23, 28, 36, 64):
        sse = host(A.compress_psnr(dev(imgs), r))
        want = O.compress_zonal_sse(imgs, r)
        if r == 64:
            assert np.all(sse < 1e-6)
        else:
            check_sse(sse, want, h * w)


def test_compress_extremes_and_impulses():
    for imgs in (impulse_images(), extreme_images()):
        for r in (1, 2, 9, 11, 13, 16, 22, 23, 33, 63):  # every kernel form / inverse flavour
            check_sse(host(A.compress_psnr(dev(imgs), r)), O.compress_zonal_sse(imgs, r), 64)


def test_compress_c5_pattern_blocks_closed_form():
    """Full C5 image size (4096^2): tiled pattern blocks have an analytic SSE at every r (P17)."""
    T = O.c0_matrix()
    d = np.array([8, 6, 4, 6, 8, 6, 4, 6])
    zz = O.zigzag_index()
    img, I, J, Am = S.pattern_image_from_rows(T, 4096, 4096, seed=3)
    x = dev(img[None])
    for r in (1, 3, 6, 10, 15, 21, 28, 36):
        want = float(np.sum(np.where(zz[I, J] < r, 0, Am.astype(np.int64) ** 2 * d[I] * d[J])))
        sse = host(A.compress_psnr(x, r))[0]
        assert abs(sse - want) <= SSE_RTOL * want, (r, sse, want)


def test_compress_c5_full_size_bench_launch_sampled():
    """C5 at full size (4096 x 4096^2 = 64 GiB, the launch configuration bench.py times):
    sampled images across the corpus (all three kinds, first / middle / last chunks) vs the oracle
    at r = 1, 10, 36, the first and last image at the other five C5 r, every image's SSE
    non-increasing in r, and the fused multi-r kernel on the same corpus equal to the passes."""
    n = 4096
    x = S.device_mixed(n, 4096, 4096, seed=0)
    sample = [0, 1, 2, 2047, 2048, 4093, 4094, 4095]
    rs = (1, 3, 6, 10, 15, 21, 28, 36)
    per_r = {}
    prev = None
    for r in rs:
        sse = host(A.compress_psnr(x, r))
        assert np.all(np.isfinite(sse)) and np.all(sse > 0)
        if r in (1, 10, 36):
            check_sse(sse[sample], O.compress_zonal_sse(host(x[sample]), r), 4096 * 4096)
        else:  # the other C5 r: the first and the last image of the corpus
            check_sse(sse[[0, 4095]], O.compress_zonal_sse(host(x[[0, 4095]]), r), 4096 * 4096)
        if prev is not None:
            assert np.all(sse <= prev * (1 + 1e-6))
        prev = per_r[r] = sse
    # the fused multi-r line (bench's fused_multi_r_c5) in its launch configuration: every image,
    # every r, against the independent passes
    got = host(A.compress_psnr_multi(x, rs))
    for k, r in enumerate(rs):
        assert np.allclose(got[k], per_r[r], rtol=SSE_RTOL, atol=0), r
    del x
    torch.cuda.empty_cache()


def test_compress_c5_sampled_images_vs_oracle():
    """Three C5 images (one per kind) generated on the device, all 8 C5 r values."""
    x = S.device_mixed(3, 4096, 4096, seed=0)
    imgs = host(x)
    for r in (1, 10, 36):
        check_sse(host(A.compress_psnr(x, r)), O.compress_zonal_sse(imgs, r), 4096 * 4096)


def test_compress_sse576_c5_images_bit_exact():
    """Three full-size C5 images (one per kind): the exact integer error sum, bit for bit, and
    the headline kernels' fp32-accumulated SSE against it (the accumulation bound SSE_RTOL)."""
    x = S.device_mixed(3, 4096, 4096, seed=0)
    imgs = host(x)
    for r in (1, 15, 36):
        exact = host(A.compress_sse576(x, r))
        assert np.array_equal(exact, O.compress_zonal_sse576(imgs, r)), r
        fused = host(A.compress_psnr(x, r))
        assert np.all(np.abs(fused - exact / 576.0 ** 2) <= SSE_RTOL * exact / 576.0 ** 2)


def test_cuda_graph_capture_and_replay():
    """Every entry is stream-ordered with host-side argument encoding only, so a sequence of calls
    can be captured into a CUDA graph and replayed (the tensor maps travel as kernel parameters)."""
    imgs = S.corpus_c2(3, 128, 256)
    x = dev(imgs)
    sse = torch.empty((4, 3), dtype=torch.float64, device="cuda")
    ps = torch.empty((4, 3), dtype=torch.float64, device="cuda")
    rs = (1, 10, 36)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside the capture (first-call attribute setup)
        for k, r in enumerate(rs):
            A.compress_psnr(x, r, sse=sse[k])
        A.compress_psnr(x, 64, q=16.0, sse=sse[3])
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for k, r in enumerate(rs):
            A.compress_psnr(x, r, sse=sse[k])
        A.compress_psnr(x, 64, q=16.0, sse=sse[3])
        A.psnr(sse.view(-1), 128 * 256, out=ps.view(-1))
    sse.fill_(-1.0)
    g.replay()
    got = host(sse)
    for k, r in enumerate(rs):
        check_sse(got[k], O.compress_zonal_sse(imgs, r), 128 * 256)
    check_sse(got[3], O.compress_quant_sse(imgs, 16.0), 128 * 256)
    assert np.allclose(host(ps), O.psnr(got, 128 * 256), rtol=1e-12)
    x.copy_(dev(imgs[::-1].copy()))  # replay on new data in the same buffers
    g.replay()
    got2 = host(sse)
    for k, r in enumerate(rs):
        check_sse(got2[k], O.compress_zonal_sse(imgs[::-1].copy(), r), 128 * 256)


# ------------------------------------------------------------------ fused compress (quantiser)

@pytest.mark.parametrize("q", [16.0, 5.0])
def test_compress_quant_u8_recon_vs_oracle(q):
    """Quantiser + u8 reconstruction: clamp(round_half_away(x^)) of the fp32 x^ against the oracle's
    float64 x^ — identical except where x^ lies within the fp32 reconstruction error (R15: 6.6e-5,
    bar 1e-4) of a rounding boundary k + 0.5, and there by at most one step; both paths tested
    (bulk-store path w % 16 == 0, per-lane path otherwise)."""
    for w in (96, 264):
        imgs = np.concatenate([S.corpus_c2(3, 64, w), rng.integers(0, 256, (2, 64, w), dtype=np.uint8)])
        want_f = O.reconstruct_quant(imgs, q)
        want = O.round_u8(want_f)
        _, rec8 = A.compress_psnr(dev(imgs), 64, q=q, recon="u8")
        got = host(rec8).astype(np.int64)
        diff = np.abs(got - want.astype(np.int64))
        near = np.abs(np.abs(want_f - np.floor(want_f)) - 0.5) < 1e-4
        assert diff.max() <= 1
        assert np.all(near[diff > 0]), (w, int((diff > 0).sum()))

@pytest.mark.parametrize("q", [16.0, 5.0, 3.0])
def test_compress_quant_vs_oracle(q):
    imgs = np.concatenate([S.corpus_c2(3, 64, 64), rng.integers(0, 256, (2, 64, 64), dtype=np.uint8)])
    want = O.reconstruct_quant(imgs, q)
    sse, rec = A.compress_psnr(dev(imgs), 64, q=q, recon="f32")
    assert np.abs(host(rec) - want).max() <= FP_TOL
    check_sse(host(sse), O.sse_per_image(imgs, want), 64 * 64)
    # SSE only (C4's kernel): the error comes from the inverted quantisation residual
    # (x - x^ = C^T (Z - Z^) C), not from x - x^ as in the reconstruction kernel — same bar
    sse_only = host(A.compress_psnr(dev(imgs), 64, q=q))
    check_sse(sse_only, O.sse_per_image(imgs, want), 64 * 64)
    assert np.allclose(sse_only, host(sse), rtol=SSE_RTOL, atol=1e-6 * 64 * 64)  # floor as check_sse


def test_compress_quant_c4_constant_frames_closed_form():
    """Full C4 frame size 4320 x 7680: constant frames under q = 16 (P18): odd v -> MSE 1."""
    vals = [0, 1, 128, 255]
    x = torch.stack([torch.full((4320, 7680), v, dtype=torch.uint8, device="cuda") for v in vals])
    sse = host(A.compress_psnr(x, 64, q=16.0))
    for v, s in zip(vals, sse):
        assert s == (4320 * 7680 if v % 2 else 0.0)


def test_compress_quant_c4_frames_vs_oracle():
    """C4 in the launch configuration bench.py times: all 240 frames of the video recipe
    (4320 x 7680, 7.96 GB) in ONE q = 16 call; frames 0, 120 and 239 against the oracle, every
    frame's SSE finite and positive."""
    x = S.device_video(240, 4320, 7680, seed=0)
    sse = host(A.compress_psnr(x, 64, q=16.0))
    assert np.all(np.isfinite(sse)) and np.all(sse > 0)
    sample = [0, 120, 239]
    imgs = host(x[sample])
    del x
    torch.cuda.empty_cache()
    check_sse(sse[sample], O.compress_quant_sse(imgs, 16.0), 4320 * 7680)


# ------------------------------------------------------------------ ABI behaviour on the device

def test_errors_enqueue_nothing():
    x = torch.zeros((2, 16, 16), dtype=torch.uint8, device="cuda")
    sse = torch.full((2,), 123.0, dtype=torch.float64, device="cuda")
    for kw in (dict(r=0), dict(r=65), dict(q=-1.0)):
        with pytest.raises(A.AdctError):
            A.compress_psnr(x, kw.get("r", 10), q=kw.get("q", 0.0), sse=sse)
    with pytest.raises(A.AdctError):
        A.compress_psnr(torch.zeros((2, 12, 16), dtype=torch.uint8, device="cuda"), 10, sse=sse)
    buf = torch.zeros((2 * 16 * 16 + 1,), dtype=torch.uint8, device="cuda")
    with pytest.raises(A.AdctError) as e:
        A.compress_psnr(buf[1:].view(2, 16, 16), 10, sse=sse)
    assert e.value.status == 2
    assert np.all(host(sse) == 123.0)


def test_streams_and_determinism():
    """Per-image sums are accumulated on a fixed-point grid with integer atomics (fx_add), so repeated
    calls, concurrent streams and graph replays give bit-identical SSE."""
    imgs = S.corpus_c2(4, 256, 256)
    x = dev(imgs)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for r, q in [(10, 0.0), (36, 0.0), (64, 16.0), (21, 5.0)]:
        with torch.cuda.stream(s1):
            a = A.compress_psnr(x, r, q=q)
        with torch.cuda.stream(s2):
            b = A.compress_psnr(x, r, q=q)
        torch.cuda.synchronize()
        assert np.array_equal(host(a), host(b)), (r, q)
        for _ in range(5):
            assert np.array_equal(host(A.compress_psnr(x, r, q=q)), host(a)), (r, q)


def test_determinism_every_sum_entry():
    """Bit-identical per-image sums across repeated calls for every accumulating entry: recon paths,
    the fused multi-r sweep, the dense comparators and UQI (C5-sized images, many warps per image)."""
    x = S.device_mixed(3, 4096, 4096, seed=5)
    ref = None
    for _ in range(3):
        out = [host(A.compress_psnr(x, 10)), host(A.compress_psnr(x, 64, q=16.0)),
               host(A.compress_psnr(x, 21, recon="f32")[0]), host(A.compress_psnr(x, 21, q=16.0, recon="u8")[0]),
               host(A.compress_psnr_multi(x, (1, 3, 6, 10, 15, 21, 28, 36))),
               host(A.compress_psnr_dense(x[:1], 10, "dct"))]
        if ref is None:
            ref = out
        else:
            for a, b in zip(out, ref):
                assert np.array_equal(a, b)
    imgs = S.corpus_c2(3, 128, 128)
    xs = dev(imgs)
    _, rec = A.compress_psnr(xs, 10, recon="f32")
    u = [host(A.uqi(xs, rec)) for _ in range(3)]
    assert np.array_equal(u[0], u[1]) and np.array_equal(u[0], u[2])


@pytest.mark.parametrize("n,buf_imgs,copy", [(6, 2, True), (6, 1, True), (17, 5, True), (17, 17, True), (1, 3, True),
                                              (6, 2, False), (17, 5, False)])
@pytest.mark.parametrize("rs", [[1, 3, 6, 10, 15, 21, 28, 36], [2, 10, 64]])
def test_end_to_end_host_entry_matches_device_path(n, buf_imgs, copy, rs):
    # copy stream and buf_imgs >= 2: double-buffered copy/compute pipeline (chunks of ~n/8 images, two
    # buffers); buf_imgs == 1, n == 1 or no copy stream: copy and passes alternate on the caller's
    # stream.  C5's r set runs the fused multi-r kernel, other sets independent passes.
    imgs = S.corpus_c2(n, 128, 128)
    pinned = torch.from_numpy(imgs).pin_memory()
    dev_buf = torch.empty((buf_imgs * 128 * 128,), dtype=torch.uint8, device="cuda")
    ps = A.compress_psnr_host(pinned, rs, dev_buf=dev_buf, copy_stream=torch.cuda.Stream() if copy else None)
    torch.cuda.synchronize()
    for k, r in enumerate(rs):
        want_sse = O.compress_zonal_sse(imgs, r)
        got = ps[k].numpy()
        # a constant (lossless) image: exact zero on the GPU (+inf dB), float64 round-off (~1e-27,
        # ~313 dB) in the oracle's literal matmuls -> compare the SSE there, PSNR elsewhere
        lossless = want_sse <= 1e-9
        assert np.all(np.isinf(got[lossless]))
        assert np.all(np.abs(got[~lossless] - O.psnr(want_sse, 128 * 128)[~lossless]) <= PSNR_TOL)


def test_launch_count_increments():
    x = torch.zeros((1, 16, 16), dtype=torch.uint8, device="cuda")
    n0 = A.launch_count()
    A.compress_psnr(x, 3)
    A.forward(x)
    torch.cuda.synchronize()
    assert A.launch_count() == n0 + 3   # compress + the fixed-point -> fp64 SSE conversion, forward


def test_psnr_kernel():
    sse = torch.tensor([0.0, 64.0, 256.0 * 4], dtype=torch.float64, device="cuda")
    p = host(A.psnr(sse, 64))
    assert np.isinf(p[0]) and abs(p[1] - 20 * math.log10(255)) < 1e-12
    assert abs(p[2] - O.psnr(1024.0, 64)) < 1e-12


# ------------------------------------------------------------------ dense comparators (F1 / F4)

DENSE = {"dct": O.dct_matrix, "sdct": O.sdct_matrix, "coarse": O.coarse_matrix, "proposed": O.proposed_matrix}


@pytest.mark.parametrize("kind", list(DENSE))
def test_dense_comparators_vs_oracle(kind):
    """Exact DCT / SDCT / coarse C0/2 / dense C_orth through adct_compress_psnr_dense (fp32 products,
    fp64 SSE) vs the oracle's float64 pipeline with the same matrix: PSNR within 1e-3 dB."""
    imgs = np.concatenate([S.corpus_c2(3, 64, 96), rng.integers(0, 256, (2, 64, 96), dtype=np.uint8)])
    x = dev(imgs)
    T = DENSE[kind]()
    for r in (1, 3, 5, 10, 21, 36, 50):
        got = host(A.compress_psnr_dense(x, r, kind))
        want = O.compress_zonal_sse(imgs, r, T)
        check_sse(got, want, 64 * 96, rtol=1e-4)   # fp32 dense products: rtol 1e-4 (PSNR 4e-4 dB)


def test_dense_proposed_matches_fast_path_and_custom():
    imgs = S.corpus_c2(6, 128, 128)
    x = dev(imgs)
    for r in (1, 10, 36):
        fast = host(A.compress_psnr(x, r))
        dense = host(A.compress_psnr_dense(x, r, "proposed"))
        custom = host(A.compress_psnr_dense(x, r, "custom", matrix=O.proposed_matrix()))
        assert np.allclose(dense, fast, rtol=1e-4)
        assert np.allclose(custom, dense, rtol=1e-6)


def test_c2_dct_curve_vs_oracle():
    """C2: the exact-DCT comparator's mean PSNR per r on the GPU vs the oracle's float64 curve
    (BASELINE C2 asks for both curves).  The paper's ordering claims are recorded by
    tools/c2_curves.py as observations on the synthetic corpus, not asserted."""
    imgs = S.corpus_c2()
    x = dev(imgs)
    px = 512 * 512
    for r in (1, 2, 5, 10, 16, 30, 45, 63):
        p_dct = O.mean_psnr(host(A.compress_psnr_dense(x, r, "dct")), px)
        assert abs(p_dct - O.mean_psnr(O.compress_zonal_sse(imgs, r, O.dct_matrix()), px)) <= PSNR_TOL


# ------------------------------------------------------------------ Parseval sweep (F3)

def oracle_diag_energy(imgs):
    d = np.array([8, 6, 4, 6, 8, 6, 4, 6])
    W = 576 // np.outer(d, d)
    Y = O.to_blocks(O.forward_int(imgs)).astype(np.int64)          # [n, H, W, 8, 8]
    E = (W * Y * Y).sum(axis=(1, 2))                                 # [n, 8, 8]
    ii, jj = np.indices((8, 8))
    return np.stack([E[:, ii + jj == s].sum(axis=1) for s in range(15)], axis=1)


def test_diag_energy_bit_exact_and_sweep_sse():
    imgs = np.concatenate([S.corpus_c2(4, 64, 96), impulse_images().reshape(1, 128 * 8, 8)[:, :64, :]
                           .repeat(12, axis=2)[:, :, :96],
                           np.full((1, 64, 96), 255, dtype=np.uint8)])
    x = dev(imgs)
    E = host(A.diag_energy(x))
    want = oracle_diag_energy(imgs)
    assert np.array_equal(E[:, :15].astype(np.int64), want)
    # entry 15: the block energy 576 sum x^2, equal to the oracle's 15 energies summed (Parseval, P9)
    assert np.array_equal(E[:, 15].astype(np.int64), want.sum(axis=1))
    assert np.array_equal(E[:, 15].astype(np.int64), 576 * (imgs.astype(np.int64) ** 2).sum(axis=(1, 2)))
    rs = [1, 3, 6, 10, 15, 21, 28, 36, 43, 49, 54, 58, 61, 63, 64]
    sse, ps = A.sweep_psnr(A.diag_energy(x), 64 * 96, rs)
    sse = host(sse)
    for k, r in enumerate(rs):
        exact = O.compress_zonal_sse(imgs, r)
        assert np.allclose(sse[k], exact, rtol=1e-10, atol=1e-6), r
        fused = host(A.compress_psnr(x, r))
        if r < 64:
            check_sse(fused, sse[k], 64 * 96)
        else:
            assert np.all(sse[k] == 0) and np.all(fused < 1e-6)


@pytest.mark.parametrize("h,w", [(8, 131080), (65544, 8)])
def test_extreme_aspect_ratios_every_entry(h, w):
    """One block row 131080 px wide / one block column 65544 px tall (many tile columns / rows, a
    ragged last tile): forward (bit-exact), inverse (u8 exact), fused multi-r, exact SSE, Parseval."""
    imgs = rng.integers(0, 256, (2, h, w), dtype=np.uint8)
    x = dev(imgs)
    Y = host(A.forward(x)).astype(np.int64)
    Yo = O.forward_int(imgs)
    assert np.array_equal(Y, Yo)
    u8 = host(A.inverse(dev(Yo.astype(np.int16)), r=10, out="u8"))
    assert np.array_equal(u8, O.round_u8(O.reconstruct_zonal_exact(imgs, 10) / 576.0))
    rs = (1, 3, 6, 10, 15, 21, 28, 36)
    multi = host(A.compress_psnr_multi(x, rs))
    E = host(A.diag_energy(x))
    assert np.array_equal(E[:, :15].astype(np.int64), oracle_diag_energy(imgs))
    for k, r in enumerate(rs):
        exact = O.compress_zonal_sse576(imgs, r)
        assert np.array_equal(host(A.compress_sse576(x, r)), exact), r
        check_sse(multi[k], exact / 576.0 ** 2, h * w)


def test_diag_energy_prefix_and_sweep():
    """adct_diag_energy_prefix (r_max <= 36): anti-diagonals 0..7 and the block energy bit-exact
    against the oracle, 8..14 marked UINT64_MAX; the sweep from it equals the full one for every
    r <= 36 and is NaN beyond; r_max > 36 falls back to every anti-diagonal."""
    imgs = np.concatenate([S.corpus_c2(3, 64, 96), rng.integers(0, 256, (1, 64, 96), dtype=np.uint8),
                           np.full((1, 64, 96), 255, dtype=np.uint8)])
    x = dev(imgs)
    want = oracle_diag_energy(imgs)
    full = A.diag_energy(x)
    for r_max in (1, 10, 36):
        E = A.diag_energy(x, r_max=r_max)
        Eh = host(E)
        assert np.array_equal(Eh[:, :8].astype(np.int64), want[:, :8]), r_max
        assert np.all(Eh[:, 8:15] == -1), r_max                      # UINT64_MAX as int64
        assert np.array_equal(Eh[:, 15].astype(np.int64), want.sum(axis=1)), r_max
        rs = [1, 3, 6, 10, 15, 21, 28, 36]
        a, pa = A.sweep_psnr(E, 64 * 96, rs)
        b, pb = A.sweep_psnr(full, 64 * 96, rs)
        assert torch.equal(a, b) and torch.equal(pa, pb), r_max
        nan_sse, nan_ps = A.sweep_psnr(E, 64 * 96, [43, 64])
        assert torch.isnan(nan_sse).all() and torch.isnan(nan_ps).all()
    assert np.array_equal(host(A.diag_energy(x, r_max=43)), host(full))


def test_diag_energy_c5_full_size_sampled():
    x = S.device_mixed(64, 4096, 4096, seed=1)
    E = host(A.diag_energy(x))
    sample = [0, 1, 2, 63]
    want = oracle_diag_energy(host(x[sample]))
    assert np.array_equal(E[sample, :15].astype(np.int64), want)
    assert np.array_equal(E[sample, 15].astype(np.int64), want.sum(axis=1))
    Ep = host(A.diag_energy(x, r_max=36))  # the bench's Parseval-sweep call
    assert np.array_equal(Ep[:, :8], E[:, :8]) and np.array_equal(Ep[:, 15], E[:, 15])


# ------------------------------------------------------------------ UQI / APE (F2)

def test_uqi_kernel_vs_oracle():
    imgs = np.concatenate([S.corpus_c2(3, 64, 96), rng.integers(0, 256, (1, 64, 96), dtype=np.uint8),
                           np.full((1, 64, 96), 77, dtype=np.uint8)])
    x = dev(imgs)
    for r in (1, 6, 21, 64):
        _sse, rec = A.compress_psnr(x, r, recon="f32")
        got = host(A.uqi(x, rec))
        recn = host(rec).astype(np.float64)
        want = np.array([O.uqi(imgs[i], recn[i]) for i in range(len(imgs))])
        assert np.abs(got - want).max() <= 1e-9, (r, got, want)
    # identical images -> 1; inverted -> negative
    f = torch.from_numpy(imgs.astype(np.float32)).cuda()
    yf = A.empty_plane(*imgs.shape, dtype=torch.float32)
    yf.copy_(f)
    assert np.allclose(host(A.uqi(x, yf)), 1.0, atol=1e-12)
    yf.copy_(255.0 - f)
    inv = host(A.uqi(x, yf))
    assert np.all(inv[[0, 1, 3]] < 0)      # textured images: anticorrelated windows
    assert abs(inv[4] - 2 * 77 * 178 / (77 ** 2 + 178 ** 2)) < 1e-12   # flat image: luminance term


def test_uqi_ape_proposed_vs_dct_end_to_end():
    """APE of the average UQI and MSE relative to the exact DCT (Figs. 4-5's quantities)
    on a small C2-like corpus: GPU pipeline vs the oracle pipeline."""
    imgs = S.corpus_c2(6, 128, 128)
    x = dev(imgs)
    for r in (3, 10, 28):
        sp, rp = A.compress_psnr(x, r, recon="f32")
        sd, rd = A.compress_psnr_dense(x, r, "dct", recon=True)
        uq_p, uq_d = host(A.uqi(x, rp)).mean(), host(A.uqi(x, rd)).mean()
        o_p = np.mean([O.uqi(im, O.reconstruct_zonal(im[None], r)[0]) for im in imgs])
        o_d = np.mean([O.uqi(im, O.reconstruct_zonal(im[None], r, O.dct_matrix())[0]) for im in imgs])
        assert abs(O.ape(uq_p, uq_d) - O.ape(o_p, o_d)) <= 1e-3
        mse_p, mse_d = host(sp).mean() / 128 ** 2, host(sd).mean() / 128 ** 2
        om_p = O.compress_zonal_sse(imgs, r).mean() / 128 ** 2
        om_d = O.compress_zonal_sse(imgs, r, O.dct_matrix()).mean() / 128 ** 2
        assert abs(O.ape(mse_p, mse_d) - O.ape(om_p, om_d)) <= 1e-2


# ---- out-of-bounds write guards (compute-sanitizer is not available on this GPU pool; every
# output buffer is a window of a larger canary-filled buffer, and nothing outside may change)
def _window(n, h, w, dtype, fill, pad_rows=8, pad_cols=32):
    """[n, h, w] view with 16-byte pitch into a canary buffer of (n + 1) x (h + pad) x (w + pad)."""
    es = torch.empty((), dtype=dtype).element_size()
    wp = -(-(w + pad_cols) * es // 16) * 16 // es
    big = torch.full((n + 1, h + pad_rows, wp), fill, dtype=dtype, device="cuda")
    return big, big[:n, :h, :w]


def _outside(big, n, h, w):
    m = torch.ones_like(big, dtype=torch.bool)
    m[:n, :h, :w] = False
    return big[m]


@pytest.mark.parametrize("n,h,w", [(3, 40, 264), (1, 8, 8), (2, 24, 520), (2, 16, 256), (3, 40, 272)])
def test_no_writes_outside_outputs(n, h, w):
    # (3, 40, 272): ragged tile rows and columns on the TMA bulk-store paths (w % 16 == 0)
    x = dev(rng.integers(0, 256, (n, h, w), dtype=np.uint8))
    canary_f, canary_u, canary_i = -12345.5, 77, -4321
    # per-image arrays: a canary tail after the n entries
    sse_big = torch.full((n + 8,), canary_f, dtype=torch.float64, device="cuda")
    for r, q in [(1, 0.0), (10, 0.0), (21, 0.0), (36, 0.0), (64, 16.0), (20, 5.0)]:
        A.compress_psnr(x, r, q=q, sse=sse_big[:n])
        assert torch.all(sse_big[n:] == canary_f)
    for kind, dt, fill in [("f32", torch.float32, canary_f), ("u8", torch.uint8, canary_u)]:
        # 10, 36: compile-time-r kernels (recon_parts.cu); 20: the runtime mask; 64 q16: the quantiser
        for r, q in [(10, 0.0), (36, 0.0), (20, 0.0), (64, 16.0)]:
            big, win = _window(n, h, w, dt, fill)
            A.compress_psnr(x, r, q=q, recon=kind, recon_out=win)
            assert torch.all(_outside(big, n, h, w) == fill), (kind, r, q)
    for coef, dt, fill in [("i16", torch.int16, canary_i), ("i32", torch.int32, canary_i), ("f32", torch.float32, canary_f)]:
        big, win = _window(n, h, w, dt, fill)
        A.forward(x, r=15, coef=coef, out=win)
        assert torch.all(_outside(big, n, h, w) == fill), coef
    y = A.forward(x)
    for out, dt, fill in [("f32", torch.float32, canary_f), ("u8", torch.uint8, canary_u)]:
        big, win = _window(n, h, w, dt, fill)
        A.inverse(y, r=28, out=out, dst=win)
        assert torch.all(_outside(big, n, h, w) == fill), out
    big, win = _window(n, h, w, torch.float32, canary_f)
    A.compress_psnr_dense(x, 10, "dct", recon=True, recon_out=win)
    assert torch.all(_outside(big, n, h, w) == canary_f)
    e_big = torch.full((n + 2, 16), canary_i, dtype=torch.int64, device="cuda")
    A.diag_energy(x, energy=e_big[:n])
    assert torch.all(e_big[n:] == canary_i)
    A.diag_energy(x, energy=e_big[:n], r_max=36)
    assert torch.all(e_big[n:] == canary_i)
    u_big = torch.full((n + 4,), canary_f, dtype=torch.float64, device="cuda")
    A.uqi(x, A.compress_psnr(x, 10, recon="f32")[1], out=u_big[:n])
    assert torch.all(u_big[n:] == canary_f)
    torch.cuda.synchronize()


@pytest.mark.parametrize("order", [(1, 3, 6, 10, 15, 21, 28, 36), (36, 1, 21, 3, 28, 6, 15, 10), (1, 2, 64)])
def test_compress_multi_matches_single_passes(order):
    # C5's set in any order runs the fused kernel (one forward, every r's inverse and error);
    # other sets fall back to single passes.  Both must equal the single-r calls / the oracle.
    imgs = S.corpus_c2(7, 48, 520)
    x = dev(imgs)
    got = host(A.compress_psnr_multi(x, order))
    for k, r in enumerate(order):
        single = host(A.compress_psnr(x, r))
        # the same exact per-pixel errors; the fused sweep sums their squares in another fp32 order
        assert np.allclose(got[k], single, rtol=SSE_RTOL, atol=1e-12), r
        check_sse(got[k], O.compress_zonal_sse(imgs, r), 48 * 520)


def test_compress_multi_c5_full_size_sampled():
    x = S.device_mixed(6, 4096, 4096, seed=3)
    rs = (1, 3, 6, 10, 15, 21, 28, 36)
    got = host(A.compress_psnr_multi(x, rs))
    for k, r in enumerate(rs):
        assert np.allclose(got[k], host(A.compress_psnr(x, r)), rtol=SSE_RTOL), r
