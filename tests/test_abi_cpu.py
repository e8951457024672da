"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/adct.h declares,
and rejects bad arguments synchronously (before touching any device)."""
import ctypes
import os
import re

import pytest

import paper_1402_6034_b200 as A
from paper_1402_6034_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "adct.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adct_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = A.load()
    names = header_functions()
    assert len(names) == 19
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    assert set(_lib.SIGNATURES) == set(names)


def test_header_argument_counts_match_binding():
    src = open(os.path.join(ROOT, "include", "adct.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    for name, (_res, args) in _lib.SIGNATURES.items():
        m = re.search(name + r"\s*\(([^)]*)\)", src)
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), name


def test_status_strings_and_version():
    lib = A.load()
    assert lib.adct_status_string(0) == b"ok"
    assert b"invalid" in lib.adct_status_string(1)
    assert b"16-byte" in lib.adct_status_string(2)
    assert lib.adct_version() >= 10000


# argument validation happens before any CUDA call, so it can run without a GPU
def fwd(src=16, n=1, h=8, w=16, pitch=16, istr=128, r=64, coef=16, ct=0, cp=32, cis=256):
    return A.load().adct_forward(src, n, h, w, pitch, istr, r, coef, ct, cp, cis, None)


def test_forward_validation():
    E, AL = _lib.ADCT_EINVAL, _lib.ADCT_EALIGN
    assert fwd(n=0) == E
    assert fwd(h=12) == E
    assert fwd(w=0) == E
    assert fwd(r=0) == E and fwd(r=65) == E
    assert fwd(ct=7) == E
    assert fwd(src=0) == E
    assert fwd(pitch=8) == E          # pitch < w
    assert fwd(istr=64) == E          # img_stride < h * pitch
    assert fwd(src=17) == AL          # misaligned pointer
    assert fwd(pitch=24, istr=192) == AL
    assert fwd(cp=16) == E            # int16 coefficient row needs 32 bytes


def test_compress_validation():
    lib = A.load()
    E, AL = _lib.ADCT_EINVAL, _lib.ADCT_EALIGN
    ok = dict(src=16, n=1, h=8, w=16, pitch=16, istr=128, r=10, q=0.0, rec=0, rt=0, rp=0, ris=0, sse=64)

    def call(**kw):
        a = dict(ok, **kw)
        return lib.adct_compress_psnr(a["src"], a["n"], a["h"], a["w"], a["pitch"], a["istr"], a["r"], a["q"],
                                      a["rec"], a["rt"], a["rp"], a["ris"], a["sse"], None)
    assert call(r=0) == E
    assert call(q=-1.0) == E
    assert call(q=float("nan")) == E
    assert call(sse=0) == E
    assert call(sse=68) == AL
    assert call(rt=1, rec=0) == E     # recon requested without a buffer
    assert call(rt=5) == E
    assert call(w=20) == E


def test_inverse_and_psnr_validation():
    lib = A.load()
    E = _lib.ADCT_EINVAL
    assert lib.adct_inverse(16, 0, 1, 8, 16, 32, 256, 10, 16, 0, 64, 512, None) == E   # dst_t NONE
    assert lib.adct_inverse(16, 0, 1, 8, 16, 32, 256, 0, 16, 1, 64, 512, None) == E    # r = 0
    assert lib.adct_psnr(16, 0, 64, 32, None) == E
    assert lib.adct_psnr(16, 4, 0, 32, None) == E
    rl = (ctypes.c_int * 2)(10, 70)
    assert lib.adct_compress_psnr_host(16, 1, 8, 16, 16, 128, rl, 2, 0.0, 16, 4096, 64, 128, None, None) == E


def test_no_cpu_fallback():
    """The product path refuses CPU tensors instead of computing on the host."""
    torch = pytest.importorskip("torch")
    x = torch.zeros((1, 8, 8), dtype=torch.uint8)
    with pytest.raises(ValueError):
        A.compress_psnr(x, 10)
    with pytest.raises(ValueError):
        A.forward(x)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1402_6034_b200")
    for dirpath, _d, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_library_matrices_match_oracle():
    """The library builds its own matrices (no shared code); they must equal the oracle's."""
    import numpy as np
    import oracle as O
    assert np.abs(A.transform_matrix("dct") - O.dct_matrix()).max() < 1e-15
    assert np.abs(A.transform_matrix("proposed") - O.proposed_matrix()).max() < 1e-15
    assert np.abs(A.transform_matrix("sdct") - O.sdct_matrix()).max() < 1e-15
    assert np.abs(A.transform_matrix("coarse") - O.coarse_matrix()).max() < 1e-15
    # F4: the library's own Jacobi polar factor of ceil(2C) against the oracle's eigendecomposition
    assert np.abs(A.transform_matrix("ceil") - O.ceil_matrix()).max() < 1e-13
    with pytest.raises(A.AdctError):
        A.transform_matrix("custom")


def test_sdct_validation():
    lib = A.load()
    E = _lib.ADCT_EINVAL
    assert lib.adct_compress_psnr_sdct(16, 1, 8, 16, 16, 128, 0, 64, None) == E    # r = 0
    assert lib.adct_compress_psnr_sdct(16, 1, 8, 16, 16, 128, 65, 64, None) == E   # r = 65
    assert lib.adct_compress_psnr_sdct(16, 1, 8, 16, 16, 128, 10, 0, None) == E    # sse NULL
    assert lib.adct_compress_psnr_sdct(16, 1, 12, 16, 16, 192, 10, 64, None) == E  # h not a multiple of 8


def test_dense_validation():
    lib = A.load()
    E = _lib.ADCT_EINVAL
    assert lib.adct_compress_psnr_dense(16, 1, 8, 16, 16, 128, 0, 1, None, None, 0, 0, 64, None) == E   # r = 0
    assert lib.adct_compress_psnr_dense(16, 1, 8, 16, 16, 128, 10, 4, None, None, 0, 0, 64, None) == E  # custom, no T
    assert lib.adct_compress_psnr_dense(16, 1, 8, 16, 16, 128, 10, 9, None, None, 0, 0, 64, None) == E  # bad enum
    assert lib.adct_uqi(16, 1, 8, 16, 16, 128, 0, 64, 512, 64, None) == E                               # y NULL


def test_sweep_validation():
    lib = A.load()
    E = _lib.ADCT_EINVAL
    rl = (ctypes.c_int * 2)(1, 4)      # r = 4 does not end on a full anti-diagonal
    assert lib.adct_sweep_psnr(16, 1, 64, rl, 2, 32, 48, None) == E
    rl = (ctypes.c_int * 1)(10)
    assert lib.adct_sweep_psnr(16, 0, 64, rl, 1, 32, 48, None) == E
    assert lib.adct_diag_energy(16, 1, 8, 16, 16, 128, 0, None) == E
    for r_max in (0, 65):  # the prefix entry validates r_max before anything else
        assert lib.adct_diag_energy_prefix(16, 1, 8, 16, 16, 128, r_max, 32, None) == E


def test_multi_and_geometry_limits_validation():
    lib = A.load()
    E, AL = _lib.ADCT_EINVAL, _lib.ADCT_EALIGN
    rl = (ctypes.c_int * 3)(1, 10, 36)
    bad = (ctypes.c_int * 2)(0, 10)
    assert lib.adct_compress_psnr_multi(16, 1, 8, 16, 16, 128, rl, 0, 64, None) == E     # n_r = 0
    assert lib.adct_compress_psnr_multi(16, 1, 8, 16, 16, 128, bad, 2, 64, None) == E    # r = 0
    assert lib.adct_compress_psnr_multi(16, 1, 8, 16, 16, 128, None, 3, 64, None) == E   # no list
    assert lib.adct_compress_psnr_multi(16, 1, 8, 16, 16, 128, rl, 3, 0, None) == E      # no sse
    assert lib.adct_compress_psnr_multi(16, 1, 8, 16, 16, 128, rl, 3, 68, None) == AL    # misaligned sse
    # the device tile cursors are 32-bit: more than 2^30 tiles of 16 x 256 px in one call is rejected
    n_big = (1 << 30) // (2 * 16) + 1                                                     # 512 x 4096 images
    assert lib.adct_compress_psnr(16, n_big, 512, 4096, 4096, 512 * 4096, 10, 0.0, 0, 0, 0, 0, 64, None) == E


def test_sse576_validation():
    lib = A.load()
    E, AL = _lib.ADCT_EINVAL, _lib.ADCT_EALIGN
    assert lib.adct_compress_sse576(16, 1, 8, 16, 16, 128, 0, 64, None, None) == E     # r = 0
    assert lib.adct_compress_sse576(16, 1, 8, 16, 16, 128, 65, 64, None, None) == E    # r = 65
    assert lib.adct_compress_sse576(16, 1, 8, 16, 16, 128, 10, None, None, None) == E  # no sse576
    assert lib.adct_compress_sse576(16, 1, 8, 16, 16, 128, 10, 68, None, None) == AL   # misaligned
    assert lib.adct_compress_sse576(16, 1, 8, 16, 16, 128, 10, 64, 68, None) == AL     # misaligned sse
    assert lib.adct_compress_sse576(16, 1, 7, 16, 16, 128, 10, 64, None, None) == E    # h % 8
    # the per-image sum is bounded by 329205^2 h w < 2^63 only for h w <= 2^26: larger is rejected
    h, w = 8192, 8200
    assert lib.adct_compress_sse576(16, 1, h, w, w, h * w, 10, 64, None, None) == E


def test_header_is_plain_c99(tmp_path):
    """include/adct.h is a C ABI: it compiles as C99 (gcc) with only the CUDA headers on the path."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = tmp_path / "h.c"
    src.write_text('#include "adct.h"\nint main(void) { return (int)ADCT_OK; }\n')
    r = subprocess.run([gcc, "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                        "-I", "/usr/local/cuda/include", "-c", str(src), "-o", str(tmp_path / "h.o")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
