"""Throughput of the non-headline compress variants (runtime-mask / quantiser / reconstruction
store) and the forward / inverse kernels, for DESIGN.md.  Synthetic C5-kind images (32 x 4096^2)
and C4-shaped frames (8 x 4320 x 7680); CUDA events, best of 3 rounds of 5 launches.

    python tools/time_variants.py > profiles/r01_variants.txt
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1402_6034_b200 import _lib  # noqa: E402
if os.environ.get("ADCT_LIB"):  # time another build (tools/build_variant.py)
    _lib.LIB_PATH = os.environ["ADCT_LIB"]
    os.environ["ADCT_LENIENT_LOAD"] = "1"
import paper_1402_6034_b200 as A  # noqa: E402
from synth import images as S  # noqa: E402


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def best_ms(fn, rounds=3, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


def main():
    pk = peak()
    rows = []
    x = S.device_mixed(32, 4096, 4096, seed=0, device="cuda")
    px = x.numel()
    sse = torch.empty(32, dtype=torch.float64, device="cuda")
    rec_f = A.empty_plane(32, 4096, 4096, torch.float32)
    rec_u = A.empty_plane(32, 4096, 4096, torch.uint8)
    coef = A.empty_plane(32, 4096, 4096, torch.int16)

    def add(name, ms, bpp):
        rows.append((name, px / (ms * 1e-3) / 1e9, bpp * px / (ms * 1e-3) / 1e9 / pk, ms))

    for r in (10, 36):
        add(f"zonal r={r} SSE only (compile-time r)", best_ms(lambda: A.compress_psnr(x, r, sse=sse)), 1)
        add(f"zonal r={r} + f32 recon", best_ms(lambda: A.compress_psnr(x, r, sse=sse, recon="f32", recon_out=rec_f)), 5)
        add(f"zonal r={r} + u8 recon", best_ms(lambda: A.compress_psnr(x, r, sse=sse, recon="u8", recon_out=rec_u)), 2)
    s576 = torch.empty(32, dtype=torch.int64, device="cuda")
    add("zonal r=10 exact u64 SSE (adct_compress_sse576)", best_ms(lambda: A.compress_sse576(x, 10, sse576=s576)), 1)
    add("quant q=16 SSE only", best_ms(lambda: A.compress_psnr(x, 64, q=16.0, sse=sse)), 1)
    add("quant q=16 + u8 recon", best_ms(lambda: A.compress_psnr(x, 64, q=16.0, sse=sse, recon="u8", recon_out=rec_u)), 2)
    add("quant q=16 r=36 SSE only (runtime mask)", best_ms(lambda: A.compress_psnr(x, 36, q=16.0, sse=sse)), 1)
    add("quant q=16 + f32 recon", best_ms(lambda: A.compress_psnr(x, 64, q=16.0, sse=sse, recon="f32", recon_out=rec_f)), 5)
    if hasattr(A.load(), "adct_compress_psnr_sdct"):
        add("SDCT integer fast path r=10", best_ms(lambda: A.compress_psnr_sdct(x, 10, sse=sse)), 1)
    add("dense exact DCT r=10", best_ms(lambda: A.compress_psnr_dense(x, 10, "dct", sse=sse)), 1)
    en = torch.empty(32 * 16, dtype=torch.int64, device="cuda")
    add("Parseval diag energy (forward + anti-diagonal energies)", best_ms(lambda: A.diag_energy(x, energy=en)), 1)
    msm = best_ms(lambda: A.compress_psnr_multi(x, (1, 3, 6, 10, 15, 21, 28, 36)))
    rows.append(("fused multi-r sweep (8 r, Gpix-passes/s)", 8 * px / (msm * 1e-3) / 1e9, px / (msm * 1e-3) / 1e9 / pk, msm))
    add("forward int16 (r=64)", best_ms(lambda: A.forward(x, out=coef)), 3)
    add("inverse int16 -> f32 (r=64)", best_ms(lambda: A.inverse(coef, r=64, out="f32", dst=rec_f)), 6)
    del x, rec_f, rec_u, coef
    v = S.device_video(8, 4320, 7680, seed=0, device="cuda")
    pxv = v.numel()
    ssev = torch.empty(8, dtype=torch.float64, device="cuda")
    ms = best_ms(lambda: A.compress_psnr(v, 64, q=16.0, sse=ssev))
    rows.append(("C4 frames 8 x 4320x7680 quant q=16 SSE only", pxv / (ms * 1e-3) / 1e9, pxv / (ms * 1e-3) / 1e9 / pk, ms))
    print(f"# {os.environ.get('ADCT_LIB', 'default build')}")
    print(f"# variants on one B200 (32 x 4096^2 C5-kind images unless noted); HBM fraction of {pk:.0f} GB/s "
          f"at the algorithmic bytes/px (1 read + output)")
    print(f"{'variant':48s} {'Gpix/s':>9s} {'HBM frac':>9s} {'ms':>9s}")
    for name, g, f, ms in rows:
        print(f"{name:48s} {g:9.1f} {f:9.3f} {ms:9.3f}")


if __name__ == "__main__":
    main()
