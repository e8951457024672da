"""C2 curves on the GPU (BASELINE configs[1]): per r = 1..64 over the 45 synthetic 512x512
images, for the proposed transform (fused fast path), the exact DCT and the SDCT (dense comparator
path; the SDCT SSE also from its integer fast path, column sdct_fast_psnr) and the F4 ceil variant
(dense): average MSE, PSNR and UQI, and the absolute percentage errors of average MSE and UQI vs the
exact DCT (the quantities of the paper's Figs. 3-5).
Writes CSV (transform,r,avg_mse,avg_psnr,avg_uqi,ape_mse,ape_uqi) to stdout or --out."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1402_6034_b200 as A  # noqa: E402
from synth import images as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
a = ap.parse_args()
imgs = S.corpus_c2()
x = A.to_device(imgs)
px = 512 * 512
rows = ["transform,r,avg_mse,avg_psnr,avg_uqi,ape_mse,ape_uqi,sdct_fast_psnr"]
for r in range(1, 65):
    sp, rp = A.compress_psnr(x, r, recon="f32")
    sd, rd = A.compress_psnr_dense(x, r, "dct", recon=True)
    ss, rs = A.compress_psnr_dense(x, r, "sdct", recon=True)
    sc, rc = A.compress_psnr_dense(x, r, "ceil", recon=True)
    sf = A.compress_psnr_sdct(x, r).cpu().numpy() / px
    with np.errstate(divide="ignore"):
        fast_psnr = float(np.mean(np.where(sf > 0, 10 * np.log10(255.0 ** 2 / np.where(sf > 0, sf, 1)), np.inf)))
    res = {"proposed": (sp, A.uqi(x, rp)), "dct": (sd, A.uqi(x, rd)), "sdct": (ss, A.uqi(x, rs)),
           "ceil": (sc, A.uqi(x, rc))}
    torch.cuda.synchronize()
    vals = {k: (v[0].cpu().numpy() / px, v[1].cpu().numpy()) for k, v in res.items()}
    ref_mse, ref_uqi = vals["dct"][0].mean(), vals["dct"][1].mean()
    for k, (m, u) in vals.items():
        with np.errstate(divide="ignore"):
            psnr = np.where(m > 0, 10 * np.log10(255.0 ** 2 / np.where(m > 0, m, 1)), np.inf)
        ape_m = 100 * abs(m.mean() - ref_mse) / ref_mse if ref_mse > 0 else 0.0
        ape_u = 100 * abs(u.mean() - ref_uqi) / abs(ref_uqi)
        extra = f"{fast_psnr:.6f}" if k == "sdct" else ""
        rows.append(f"{k},{r},{m.mean():.6f},{np.mean(psnr):.6f},{u.mean():.8f},{ape_m:.4f},{ape_u:.5f},{extra}")
txt = "\n".join(rows) + "\n"
if a.out:
    open(a.out, "w").write(txt)
print(txt)
