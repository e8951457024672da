"""Seeded synthetic 8-bit greyscale inputs shaped like the paper's workloads.

This module holds NO arithmetic of the method (no transform, mask, quantiser or metric);
it only draws images.  It is the one module shared by the oracle-side tests and the
product-side bench (DESIGN.md §4 states the recipe).  The paper's own corpus (45 USC-SIPI
512x512 8-bit images) is not available; these generators stand in for it.

Host generators (numpy PCG64) serve the small configs C1/C2 and tests; device generators
(torch, CUDA) serve the large configs C3-C5.  Host and device generators follow the same
recipe but are NOT bit-identical: the oracle always consumes the exact bytes the GPU
consumed (copied back), so no cross-device reproducibility is needed.
"""
from __future__ import annotations

import math

import numpy as np

KIND_SMOOTH, KIND_TEXTURED, KIND_RECTS = 0, 1, 2


# ----------------------------------------------------------------------------- host (numpy)

def _sinusoid_field(rng: np.random.Generator, h: int, w: int, n_waves: int = 8) -> np.ndarray:
    """128 + sum_k A_k sin(2 pi (fx_k x + fy_k y) + phi_k); f ~ U[0, 0.1] cyc/px, A_k ~ U[4, 16]."""
    y = np.arange(h, dtype=np.float64)[:, None]
    x = np.arange(w, dtype=np.float64)[None, :]
    f = 128.0 + np.zeros((h, w))
    for _ in range(n_waves):
        fx, fy = rng.uniform(0.0, 0.1, size=2)
        phi = rng.uniform(0.0, 2 * math.pi)
        amp = rng.uniform(4.0, 16.0)
        f += amp * np.sin(2 * math.pi * (fx * x + fy * y) + phi)
    return f


def _rects(rng: np.random.Generator, h: int, w: int, n_rects: int = 24, side=(16, 256)) -> np.ndarray:
    """Piecewise-constant: background U{0..255}, n_rects rectangles (painter's order)."""
    img = np.full((h, w), rng.integers(0, 256), dtype=np.float64)
    for _ in range(n_rects):
        rh, rw = rng.integers(side[0], side[1] + 1, size=2)
        y0 = rng.integers(0, max(1, h - rh + 1))
        x0 = rng.integers(0, max(1, w - rw + 1))
        img[y0:y0 + rh, x0:x0 + rw] = rng.integers(0, 256)
    return img


def _to_u8(f: np.ndarray) -> np.ndarray:
    return np.clip(np.rint(f), 0, 255).astype(np.uint8)


def image_c1(seed: int = 0, h: int = 512, w: int = 512) -> np.ndarray:
    """BASELINE C1: smooth sinusoid sum + N(0, 8^2) noise, clipped to [0, 255]."""
    rng = np.random.default_rng(seed)
    f = _sinusoid_field(rng, h, w)
    f += rng.normal(0.0, 8.0, size=(h, w))
    return _to_u8(f)


def image_kind(seed: int, kind: int, h: int = 512, w: int = 512, rect_scale: int = 1) -> np.ndarray:
    """One image of the C2/C5 mix: 0 smooth (as C1), 1 textured (N(0, 25^2)), 2 rectangles."""
    if kind == KIND_SMOOTH:
        return image_c1(seed, h, w)
    rng = np.random.default_rng(seed)
    if kind == KIND_TEXTURED:
        f = _sinusoid_field(rng, h, w)
        f += rng.normal(0.0, 25.0, size=(h, w))
        return _to_u8(f)
    if kind == KIND_RECTS:
        return _to_u8(_rects(rng, h, w, side=(16 * rect_scale, 256 * rect_scale)))
    raise ValueError(kind)


def corpus_c2(n: int = 45, h: int = 512, w: int = 512) -> np.ndarray:
    """BASELINE C2: 45 images, seeds 0..44, kind = seed mod 3. uint8 [n, h, w]."""
    return np.stack([image_kind(s, s % 3, h, w) for s in range(n)])


def uniform_images(n: int, h: int, w: int, seed: int = 0) -> np.ndarray:
    """i.i.d. U{0..255} pixels (BASELINE C3 recipe), host version."""
    return np.random.default_rng(seed).integers(0, 256, size=(n, h, w), dtype=np.uint8)


def pattern_image_from_rows(rows: np.ndarray, h: int, w: int, amps=(1, 37, 127), seed: int = 0):
    """Tiled pattern blocks: block (by, bx) = 128 + a * outer(rows[i], rows[j]).

    (i, j, a) are drawn per block; the caller passes the rows (the tests pass C0's rows,
    so this module carries no transform constants).  Returns (img uint8 [h, w], I, J, A).
    """
    rng = np.random.default_rng(seed)
    H, W = h // 8, w // 8
    I = rng.integers(0, 8, size=(H, W))
    J = rng.integers(0, 8, size=(H, W))
    A = np.asarray(amps)[rng.integers(0, len(amps), size=(H, W))]
    rows = np.asarray(rows, dtype=np.int64)
    blocks = 128 + A[..., None, None] * rows[I][..., :, None] * rows[J][..., None, :]
    img = blocks.transpose(0, 2, 1, 3).reshape(h, w)
    assert img.min() >= 0 and img.max() <= 255
    return img.astype(np.uint8), I, J, A


# ----------------------------------------------------------------------------- device (torch)

def _torch():
    import torch
    return torch


def device_uniform(n: int, h: int, w: int, seed: int = 0, device="cuda"):
    """C3: i.i.d. U{0..255} uint8 [n, h, w] drawn on the device (chunked)."""
    torch = _torch()
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty((n, h, w), dtype=torch.uint8, device=device)
    chunk = max(1, (1 << 28) // (h * w))
    for i in range(0, n, chunk):
        j = min(n, i + chunk)
        out[i:j] = torch.randint(0, 256, (j - i, h, w), generator=g, device=device, dtype=torch.uint8)
    return out


def _device_sinusoid_field(torch, rng: np.random.Generator, h: int, w: int, device):
    """128 + sum of 8 sinusoids (parameters from the host rng) as a rank-16 product on the device."""
    fx, fy = rng.uniform(0.0, 0.1, 8), rng.uniform(0.0, 0.1, 8)
    ph, amp = rng.uniform(0.0, 2 * math.pi, 8), rng.uniform(4.0, 16.0, 8)
    two_pi = 2 * math.pi
    y = torch.arange(h, device=device, dtype=torch.float64)
    x = torch.arange(w, device=device, dtype=torch.float64)
    fy_t, fx_t = torch.tensor(fy, device=device), torch.tensor(fx, device=device)
    ph_t, amp_t = torch.tensor(ph, device=device), torch.tensor(amp, device=device)
    ay = two_pi * fy_t[:, None] * y[None, :] + ph_t[:, None]          # [8, h]
    bx = two_pi * fx_t[:, None] * x[None, :]                          # [8, w]
    # sin(a + b) = sin a cos b + cos a sin b
    U = torch.cat([amp_t[:, None] * torch.sin(ay), amp_t[:, None] * torch.cos(ay)], 0)  # [16, h]
    V = torch.cat([torch.cos(bx), torch.sin(bx)], 0)                                   # [16, w]
    return 128.0 + (U.t().float() @ V.float())                                         # [h, w] f32


def device_mixed(n: int, h: int, w: int, seed: int = 0, device="cuda", rect_scale: int = 8,
                 first_index: int = 0, out=None):
    """C5: images of kind (first_index + i) mod 3 (smooth / textured sigma 25 / rectangles).

    Image i depends only on (seed, first_index + i), so a rank draws its own shard without the rest.
    Shape parameters come from a per-image host rng; noise from a per-image device generator.
    """
    torch = _torch()
    if out is None:
        out = torch.empty((n, h, w), dtype=torch.uint8, device=device)
    g = torch.Generator(device=device)
    for i in range(n):
        gi = first_index + i
        rng = np.random.default_rng([seed, gi])
        kind = gi % 3
        if kind == KIND_RECTS:
            img = out[i]
            img.fill_(int(rng.integers(0, 256)))
            for _ in range(24):
                rh, rw = (min(int(v), d) for v, d in zip(rng.integers(16 * rect_scale, 256 * rect_scale + 1, 2), (h, w)))
                y0, x0 = int(rng.integers(0, h - rh + 1)), int(rng.integers(0, w - rw + 1))
                img[y0:y0 + rh, x0:x0 + rw] = int(rng.integers(0, 256))
        else:
            f = _device_sinusoid_field(torch, rng, h, w, device)
            g.manual_seed(seed * 1000003 + gi)
            sigma = 8.0 if kind == KIND_SMOOTH else 25.0
            f += sigma * torch.randn((h, w), generator=g, device=device, dtype=torch.float32)
            out[i] = f.round_().clamp_(0, 255).to(torch.uint8)
    return out


def device_video(n_frames: int, h: int = 4320, w: int = 7680, seed: int = 0, device="cuda",
                 sigma_blur: float = 24.0, margin: int = 736, first_frame: int = 0, out=None):
    """C4: smooth random field (Gaussian-blurred white noise, mean 128 / sd 40) on a
    (h + margin) x (w + margin) canvas; frame t = crop at cumulative offset o_t = o_{t-1} + (dy, dx),
    dy, dx ~ U{1, 2, 3}; + N(0, 4^2); rint + clip.  Offsets wrap modulo the margin.
    """
    torch = _torch()
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    H, W = h + margin, w + margin
    noise = torch.randn((H, W), generator=g, device=device, dtype=torch.float32)
    fy = torch.fft.fftfreq(H, device=device)
    fx = torch.fft.rfftfreq(W, device=device)
    filt = torch.exp(-2 * (math.pi * sigma_blur) ** 2 * (fy[:, None] ** 2 + fx[None, :] ** 2))
    field = torch.fft.irfft2(torch.fft.rfft2(noise) * filt, s=(H, W))
    field = 128.0 + 40.0 * (field - field.mean()) / field.std()
    del noise
    steps = torch.randint(1, 4, (first_frame + n_frames, 2), generator=g, device=device).cumsum(0) % margin
    if out is None:
        out = torch.empty((n_frames, h, w), dtype=torch.uint8, device=device)
    gn = torch.Generator(device=device)
    for t in range(n_frames):
        oy, ox = steps[first_frame + t].tolist()
        gn.manual_seed(seed * 7919 + first_frame + t)
        f = field[oy:oy + h, ox:ox + w] + 4.0 * torch.randn((h, w), generator=gn, device=device)
        out[t] = f.round_().clamp_(0, 255).to(torch.uint8)
    return out
