"""Interleaved A/B timing of library builds (tools/build_variant.py) in ONE process: every build is
loaded side by side (ctypes, RTLD_LOCAL) and the launches alternate build by build, so the power-capped
SM clock drifts equally over all of them (separate processes differed by up to 5 % run to run).

    python tools/ab_zonal.py [--images N] [--quant-frames F] default tune_variants/libadct_x.so ...

Per r (and C4's q = 16 quantiser on F 8K frames if requested): the median over rounds of the mean of
3 launches, as a fraction of the measured HBM bandwidth at 1 B/px; the step-equivalent harmonic mean
over C5's eight r."""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1402_6034_b200 import _lib  # noqa: E402
from synth import images as S  # noqa: E402

RS = (1, 3, 6, 10, 15, 21, 28, 36)


def load(path, entry="adct_compress_psnr"):
    lib = ctypes.CDLL(path)
    fn = getattr(lib, entry)
    fn.restype, fn.argtypes = _lib.SIGNATURES[entry]
    return fn


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=512)
    ap.add_argument("--rounds", type=int, default=7)
    ap.add_argument("--quant-frames", type=int, default=0)
    ap.add_argument("--diag", action="store_true", help="time adct_diag_energy (Parseval sweep kernel) only")
    ap.add_argument("--rs", default=None, help="comma-separated r values instead of C5's eight")
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    paths = [_lib.LIB_PATH if p == "default" else p for p in a.libs]
    fns = [load(p) for p in paths]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def bench(x, r, q):
        n, h, w = x.shape
        sse = torch.empty(n, dtype=torch.float64, device="cuda")
        args = lambda: (x.data_ptr(), n, h, w, x.stride(1), x.stride(0), r, q, None, 0, 0, 0, sse.data_ptr(), st)
        times = [[] for _ in fns]
        for fn in fns:  # warm-up
            fn(*args())
        torch.cuda.synchronize()
        for _ in range(a.rounds):
            for i, fn in enumerate(fns):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3):
                    assert fn(*args()) == 0
                e1.record()
                torch.cuda.synchronize()
                times[i].append(e0.elapsed_time(e1) / 3)
        px = x.numel()
        return [px / (statistics.median(t) * 1e-3) / 1e9 / peak for t in times]

    x = S.device_mixed(a.images, 4096, 4096, device="cuda")
    if a.diag:
        dfns = [load(p, "adct_diag_energy") for p in paths]
        n = x.shape[0]
        en = torch.empty((n, 16), dtype=torch.int64, device="cuda")
        times = [[] for _ in dfns]
        call = lambda fn: fn(x.data_ptr(), n, 4096, 4096, x.stride(1), x.stride(0), en.data_ptr(), st)
        for fn in dfns:
            call(fn)
        torch.cuda.synchronize()
        ref = en.clone()
        for _ in range(a.rounds):
            for i, fn in enumerate(dfns):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3):
                    assert call(fn) == 0
                e1.record()
                torch.cuda.synchronize()
                times[i].append(e0.elapsed_time(e1) / 3)
                assert torch.equal(en, ref), "energies differ between builds"
        for i, p in enumerate(a.libs):
            print(f"{os.path.basename(p):24s} diag energy HBM frac {x.numel() / (statistics.median(times[i]) * 1e-3) / 1e9 / peak:.4f}")
        return
    rs = tuple(int(v) for v in a.rs.split(",")) if a.rs else RS
    fr = {r: bench(x, r, 0.0) for r in rs}
    del x
    for i, p in enumerate(a.libs):
        tot = len(rs) / sum(1 / fr[r][i] for r in rs)
        print(f"{os.path.basename(p):24s} step-equivalent {tot:.4f} | " + " ".join(f"r{r}:{fr[r][i]:.3f}" for r in rs))
    if a.quant_frames:
        v = S.device_video(a.quant_frames, 4320, 7680, seed=0, device="cuda")
        fq = bench(v, 64, 16.0)
        for i, p in enumerate(a.libs):
            print(f"{os.path.basename(p):24s} C4 quant q=16 HBM frac {fq[i]:.4f}")


if __name__ == "__main__":
    main()
