"""Thin ctypes binding over libadct.so (include/adct.h).

Argument marshalling only: every step of the path runs in the library's sm_100a kernels.
torch supplies device memory and the current CUDA stream.  There is no CPU fallback: if the
library is missing or no CUDA device is present the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libadct.so")

ADCT_OK, ADCT_EINVAL, ADCT_EALIGN, ADCT_ECUDA = 0, 1, 2, 3
COEF = {"i16": 0, "i32": 1, "f32": 2}
RECON = {None: 0, "none": 0, "f32": 1, "u8": 2}

# exported symbols and their C signatures (checked by tests/test_abi_cpu.py against adct.h)
_i64, _i32, _vp, _f32 = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_float
SIGNATURES = {
    "adct_forward": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _i32, _vp, _i32, _i64, _i64, _vp]),
    "adct_inverse": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _i64, _i32, _vp, _i32, _i64, _i64, _vp]),
    "adct_compress_psnr": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _i32, _f32, _vp, _i32, _i64, _i64,
                                  _vp, _vp]),
    "adct_psnr": (_i32, [_vp, _i64, _i64, _vp, _vp]),
    "adct_compress_psnr_host": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _i32, _f32, _vp, _i64,
                                       _vp, _vp, _vp, _vp]),
    "adct_compress_psnr_multi": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _i32, _vp, _vp]),
    "adct_compress_sse576": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _vp]),
    "adct_quant_reciprocals": (_i32, [_f32, _vp]),
    "adct_compress_psnr_dense": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _i64, _i64,
                                        _vp, _vp]),
    "adct_uqi": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp]),
    "adct_transform_matrix": (_i32, [_i32, _vp]),
    "adct_diag_energy": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp]),
    "adct_diag_energy_prefix": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _i32, _vp, _vp]),
    "adct_compress_psnr_sdct": (_i32, [_vp, _i64, _i64, _i64, _i64, _i64, _i32, _vp, _vp]),
    "adct_sweep_psnr": (_i32, [_vp, _i64, _i64, _vp, _i32, _vp, _vp, _vp]),
    "adct_status_string": (ctypes.c_char_p, [_i32]),
    "adct_last_cuda_error": (_i32, []),
    "adct_version": (_i32, []),
    "adct_launch_count": (_i64, []),
}

_lib = None


class AdctError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = load().adct_status_string(status).decode()
        if status == ADCT_ECUDA:
            msg += f" (cudaError {load().adct_last_cuda_error()})"
        super().__init__(f"{where}: {msg}")


def load():
    """Load libadct.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing — run `python -m paper_1402_6034_b200.build`")
        lib = ctypes.CDLL(LIB_PATH)
        lenient = os.environ.get("ADCT_LENIENT_LOAD") == "1"  # timing older builds (tools/): skip absent entries
        for name, (res, args) in SIGNATURES.items():
            if lenient and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(st: int, where: str):
    if st != ADCT_OK:
        raise AdctError(st, where)


def _torch():
    import torch
    return torch


def _stream(stream=None):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _plane(t, elem: int):
    """(ptr, n, h, w, pitch_bytes, img_stride_bytes) of a [n, h, w] CUDA tensor with unit column stride."""
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if t.dim() != 3:
        raise ValueError("expected a [n, h, w] (or [h, w]) tensor")
    if not t.is_cuda:
        raise ValueError("tensor must be on a CUDA device (no CPU path)")
    if t.stride(2) != 1:
        raise ValueError("columns must be contiguous")
    n, h, w = t.shape
    return t.data_ptr(), n, h, w, t.stride(1) * elem, t.stride(0) * elem


def empty_plane(n: int, h: int, w: int, dtype, device="cuda"):
    """[n, h, w] tensor whose row pitch is padded to a multiple of 16 bytes (the ABI's TMA rule)."""
    torch = _torch()
    es = torch.empty((), dtype=dtype).element_size()
    wp = -(-w * es // 16) * 16 // es
    return torch.empty((n, h, wp), dtype=dtype, device=device)[:, :, :w]


def to_device(x, device="cuda"):
    """Copy a host uint8 [n, h, w] (or [h, w]) array into a 16-byte-pitched device plane."""
    torch = _torch()
    t = torch.as_tensor(np.ascontiguousarray(x) if isinstance(x, np.ndarray) else x)
    if t.dim() == 2:
        t = t.unsqueeze(0)
    out = empty_plane(*t.shape, dtype=t.dtype, device=device)
    out.copy_(t)
    return out


TRANSFORMS = {"proposed": 0, "dct": 1, "sdct": 2, "coarse": 3, "custom": 4, "ceil": 5}


def transform_matrix(kind: str) -> np.ndarray:
    """adct_transform_matrix: the library's own 8x8 matrix (host, no GPU)."""
    out = np.zeros(64, dtype=np.float64)
    _check(load().adct_transform_matrix(TRANSFORMS[kind], out.ctypes.data), "adct_transform_matrix")
    return out.reshape(8, 8)


def compress_psnr_dense(x, r: int, transform: str = "dct", matrix=None, sse=None, recon: bool = False,
                        recon_out=None, stream=None):
    """adct_compress_psnr_dense: the block pipeline with a dense 8x8 transform (comparators).

    Returns sse (float64 [n]) or (sse, recon f32 [n, h, w]) when recon=True."""
    torch = _torch()
    p, n, h, w, pitch, istr = _plane(x, 1)
    if sse is None:
        sse = torch.empty((n,), dtype=torch.float64, device=x.device)
    cm = None
    if transform == "custom":
        cm = np.ascontiguousarray(np.asarray(matrix, dtype=np.float64).reshape(64))
    rp, rpitch, ristr = None, 0, 0
    if recon:
        if recon_out is None:
            recon_out = empty_plane(n, h, w, torch.float32, x.device)
        rp, _n, _h, _w, rpitch, ristr = _plane(recon_out, 4)
    _check(load().adct_compress_psnr_dense(p, n, h, w, pitch, istr, r, TRANSFORMS[transform],
                                           cm.ctypes.data if cm is not None else None, rp, rpitch, ristr,
                                           sse.data_ptr(), _stream(stream)), "adct_compress_psnr_dense")
    return (sse, recon_out) if recon else sse


def compress_psnr_sdct(x, r: int, sse=None, stream=None):
    """adct_compress_psnr_sdct: the SDCT comparator on the integer fast path (24-add butterflies),
    per-image SSE (float64 [n], device)."""
    torch = _torch()
    p, n, h, w, pitch, istr = _plane(x, 1)
    if sse is None:
        sse = torch.empty((n,), dtype=torch.float64, device=x.device)
    _check(load().adct_compress_psnr_sdct(p, n, h, w, pitch, istr, int(r), sse.data_ptr(), _stream(stream)),
           "adct_compress_psnr_sdct")
    return sse


def uqi(x, y, out=None, stream=None):
    """adct_uqi: per-image mean UQI (8x8 sliding windows) between uint8 x and f32 y (device)."""
    torch = _torch()
    p, n, h, w, pitch, istr = _plane(x, 1)
    q, n2, h2, w2, ypitch, yistr = _plane(y, 4)
    if (n, h, w) != (n2, h2, w2):
        raise ValueError("uqi: x and y shapes differ")
    if out is None:
        out = torch.empty((n,), dtype=torch.float64, device=x.device)
    _check(load().adct_uqi(p, n, h, w, pitch, istr, q, ypitch, yistr, out.data_ptr(), _stream(stream)), "adct_uqi")
    return out


def diag_energy(x, energy=None, stream=None, r_max: int = 64):
    """adct_diag_energy (r_max = 64) / adct_diag_energy_prefix: exact per-image anti-diagonal
    energies sum W Y^2 in entries 0..14 and the block energy 576 sum x^2 in entry 15 (uint64 [n, 16],
    device); with r_max <= 36 only anti-diagonals 0..7 are computed (the others hold UINT64_MAX)."""
    torch = _torch()
    p, n, h, w, pitch, istr = _plane(x, 1)
    if energy is None:
        energy = torch.empty((n, 16), dtype=torch.int64, device=x.device)
    if r_max == 64:
        _check(load().adct_diag_energy(p, n, h, w, pitch, istr, energy.data_ptr(), _stream(stream)),
               "adct_diag_energy")
    else:
        _check(load().adct_diag_energy_prefix(p, n, h, w, pitch, istr, int(r_max), energy.data_ptr(),
                                              _stream(stream)), "adct_diag_energy_prefix")
    return energy


def sweep_psnr(energy, pixels: int, r_list, stream=None):
    """adct_sweep_psnr: (sse, psnr) [len(r_list), n] for triangular r from diag_energy's output."""
    torch = _torch()
    n = energy.shape[0]
    nr = len(r_list)
    sse = torch.empty((nr, n), dtype=torch.float64, device=energy.device)
    ps = torch.empty_like(sse)
    rl = (ctypes.c_int * nr)(*[int(v) for v in r_list])
    _check(load().adct_sweep_psnr(energy.data_ptr(), n, pixels, rl, nr, sse.data_ptr(), ps.data_ptr(),
                                  _stream(stream)), "adct_sweep_psnr")
    return sse, ps


def quant_reciprocals(q: float) -> np.ndarray:
    """adct_quant_reciprocals: the kernels' per-position quantiser constants c' (host, no GPU)."""
    out = np.zeros(64, dtype=np.float32)
    _check(load().adct_quant_reciprocals(float(q), out.ctypes.data), "adct_quant_reciprocals")
    return out.reshape(8, 8)


def launch_count() -> int:
    return int(load().adct_launch_count())


def version() -> int:
    return int(load().adct_version())


def forward(x, r: int = 64, coef: str = "i16", out=None, stream=None):
    """adct_forward: Y = T X T^T per 8x8 block (i16 / i32) or Z = D Y D (f32), image-shaped."""
    torch = _torch()
    p, n, h, w, pitch, istr = _plane(x, 1)
    dt = {"i16": torch.int16, "i32": torch.int32, "f32": torch.float32}[coef]
    if out is None:
        out = empty_plane(n, h, w, dt, x.device)
    es = out.element_size()
    q, *_rest = _plane(out, es)
    _check(load().adct_forward(p, n, h, w, pitch, istr, r, q, COEF[coef], out.stride(-2) * es,
                               out.stride(0) * es if out.dim() == 3 else h * out.stride(-2) * es,
                               _stream(stream)), "adct_forward")
    return out


def inverse(coef, r: int = 64, out: str = "f32", dst=None, stream=None):
    """adct_inverse: X^ = C^T (M_r . Z) C per block, from an image-shaped coefficient plane."""
    torch = _torch()
    kind = {torch.int16: "i16", torch.int32: "i32", torch.float32: "f32"}[coef.dtype]
    p, n, h, w, pitch, istr = _plane(coef, coef.element_size())
    if dst is None:
        dst = empty_plane(n, h, w, torch.float32 if out == "f32" else torch.uint8, coef.device)
    es = dst.element_size()
    d, *_r = _plane(dst, es)
    _check(load().adct_inverse(p, COEF[kind], n, h, w, pitch, istr, r, d, RECON[out], dst.stride(-2) * es,
                               dst.stride(0) * es if dst.dim() == 3 else h * dst.stride(-2) * es,
                               _stream(stream)), "adct_inverse")
    return dst


def compress_psnr(x, r: int, q: float = 0.0, recon: str | None = None, sse=None, recon_out=None,
                  stream=None):
    """adct_compress_psnr: fused forward + zonal (q = 0) / quantiser (q > 0) + inverse + per-image SSE.

    Returns sse (float64 [n], device) or (sse, recon) when `recon` is "f32" / "u8".
    """
    torch = _torch()
    p, n, h, w, pitch, istr = _plane(x, 1)
    if sse is None:
        sse = torch.empty((n,), dtype=torch.float64, device=x.device)
    rp, rpitch, ristr = 0, 0, 0
    if recon is not None and recon != "none":
        if recon_out is None:
            recon_out = empty_plane(n, h, w, torch.float32 if recon == "f32" else torch.uint8, x.device)
        es = recon_out.element_size()
        rp, _n, _h, _w, rpitch, ristr = _plane(recon_out, es)
    _check(load().adct_compress_psnr(p, n, h, w, pitch, istr, r, float(q), rp, RECON[recon], rpitch, ristr,
                                     sse.data_ptr(), _stream(stream)), "adct_compress_psnr")
    return (sse, recon_out) if recon not in (None, "none") else sse


def compress_psnr_multi(x, r_list, sse=None, stream=None):
    """adct_compress_psnr_multi: SSE [len(r_list), n] of the zonal pass for every r (q = 0).

    BASELINE C5's r set runs as one fused kernel (one read, one forward, every r's inverse and
    per-pixel error); other sets run independent passes."""
    torch = _torch()
    p, n, h, w, pitch, istr = _plane(x, 1)
    nr = len(r_list)
    if sse is None:
        sse = torch.empty((nr, n), dtype=torch.float64, device=x.device)
    if not sse.is_contiguous() or tuple(sse.shape) != (nr, n):
        raise ValueError("sse must be a contiguous [len(r_list), n] float64 tensor")
    rl = (ctypes.c_int * nr)(*[int(v) for v in r_list])
    _check(load().adct_compress_psnr_multi(p, n, h, w, pitch, istr, rl, nr, sse.data_ptr(), _stream(stream)),
           "adct_compress_psnr_multi")
    return sse


def compress_sse576(x, r: int, sse576=None, sse=None, stream=None):
    """adct_compress_sse576: exact per-image sum of (576 x - R)^2 as int64 [n] (zonal, q = 0).

    Bit-exact integer result (the fused kernel's fp32 accumulation is replaced by 64-bit integer
    adds).  If ``sse`` (float64 [n]) is given it also receives sse576 / 576^2.  Returns sse576
    (values < 2^63 for every accepted size, so the int64 view is exact)."""
    torch = _torch()
    p, n, h, w, pitch, istr = _plane(x, 1)
    if sse576 is None:
        sse576 = torch.empty(n, dtype=torch.int64, device=x.device)
    if sse576.dtype != torch.int64 or not sse576.is_contiguous() or sse576.numel() != n:
        raise ValueError("sse576 must be a contiguous int64 tensor of n entries")
    sp = None
    if sse is not None:
        if sse.dtype != torch.float64 or not sse.is_contiguous() or sse.numel() != n:
            raise ValueError("sse must be a contiguous float64 tensor of n entries")
        sp = sse.data_ptr()
    _check(load().adct_compress_sse576(p, n, h, w, pitch, istr, int(r), sse576.data_ptr(), sp, _stream(stream)),
           "adct_compress_sse576")
    return sse576


def psnr(sse, pixels: int, out=None, stream=None):
    """adct_psnr: 10 log10(255^2 pixels / sse), +inf where sse == 0 (device)."""
    torch = _torch()
    if out is None:
        out = torch.empty_like(sse)
    _check(load().adct_psnr(sse.data_ptr(), sse.numel(), pixels, out.data_ptr(), _stream(stream)), "adct_psnr")
    return out


def compress_psnr_host(host_images, r_list, q: float = 0.0, dev_buf=None, dev_sse=None, host_psnr=None,
                       stream=None, copy_stream=None):
    """adct_compress_psnr_host: end-to-end from host memory (pinned torch uint8 [n, h, w] or numpy).

    copy_stream: an optional torch.cuda.Stream for the overlapped (double-buffered) host->device
    copies.  Returns host PSNR [len(r_list), n] (float64, valid after the stream is synchronised).
    """
    torch = _torch()
    if isinstance(host_images, np.ndarray):
        host_images = torch.from_numpy(np.ascontiguousarray(host_images))
    if host_images.dim() == 2:
        host_images = host_images.unsqueeze(0)
    n, h, w = host_images.shape
    if host_images.is_cuda or host_images.stride(2) != 1:
        raise ValueError("host_images must be a host tensor with contiguous columns")
    dpitch = (w + 15) // 16 * 16
    if dev_buf is None:
        dev_buf = torch.empty((n * h * dpitch,), dtype=torch.uint8, device="cuda")
    nr = len(r_list)
    if dev_sse is None:
        dev_sse = torch.empty((2 * nr * n,), dtype=torch.float64, device="cuda")
    if host_psnr is None:
        host_psnr = torch.empty((nr, n), dtype=torch.float64, pin_memory=True)
    rl = (ctypes.c_int * nr)(*[int(v) for v in r_list])
    cs = ctypes.c_void_p(copy_stream.cuda_stream) if copy_stream is not None else None
    _check(load().adct_compress_psnr_host(host_images.data_ptr(), n, h, w, host_images.stride(1),
                                          host_images.stride(0), rl, nr, float(q), dev_buf.data_ptr(),
                                          dev_buf.numel(), dev_sse.data_ptr(), host_psnr.data_ptr(),
                                          _stream(stream), cs), "adct_compress_psnr_host")
    return host_psnr
