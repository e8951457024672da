"""One small launch of every kernel behind the C ABI, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_smoke.py

Small ragged shapes (partial 256-column tiles, partial 16-row tiles, odd image counts), every
compress variant (compile-time zonal direct / grouped / residual / f16 route, runtime-mask
reconstruction, quantiser), forward / inverse, dense comparator, Parseval sweep, UQI, PSNR and
the host entry.  Results are not checked here (tests/test_gpu_parity.py does that).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1402_6034_b200 as A  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    for (n, h, w) in [(3, 40, 264), (1, 8, 8), (2, 24, 520)]:
        x = A.to_device(rng.integers(0, 256, (n, h, w), dtype=np.uint8))
        for r in (1, 3, 6, 10, 15, 21, 28, 36, 50, 64):
            A.compress_psnr(x, r)
        A.compress_psnr(x, 10, recon="f32")
        A.compress_sse576(x, 10)
        A.compress_psnr(x, 36, recon="u8")
        A.compress_psnr(x, 64, q=16.0)
        A.compress_psnr(x, 20, q=5.0, recon="u8")
        y = A.forward(x)
        A.forward(x, r=10, coef="f32")
        A.inverse(y, r=28)
        A.inverse(y, r=64, out="u8")
        for kind in ("dct", "sdct"):
            A.compress_psnr_dense(x, 10, kind)
        e = A.diag_energy(x)
        A.sweep_psnr(e, h * w, (1, 3, 6, 10))
        rec = A.compress_psnr(x, 10, recon="f32")[1]
        A.uqi(x, rec)
    imgs = torch.from_numpy(rng.integers(0, 256, (5, 64, 64), dtype=np.uint8)).pin_memory()
    buf = torch.empty(2 * 64 * 64, dtype=torch.uint8, device="cuda")
    A.compress_psnr_host(imgs, [1, 10, 36], dev_buf=buf)
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
