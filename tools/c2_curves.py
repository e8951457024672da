"""C2 curves on the GPU (BASELINE configs[1]): mean PSNR per r = 1..64 over the 45 synthetic
512x512 images for the proposed transform (fused fast path), the exact DCT and the SDCT (dense
comparator path), plus MSE absolute percentage error vs the exact DCT (Fig. 5's quantity).
Writes CSV (transform,r,avg_mse,avg_psnr,ape_mse) to stdout or --out."""
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
rows = ["transform,r,avg_mse,avg_psnr,ape_mse"]
for r in range(1, 65):
    res = {"proposed": A.compress_psnr(x, r), "dct": A.compress_psnr_dense(x, r, "dct"),
           "sdct": A.compress_psnr_dense(x, r, "sdct")}
    torch.cuda.synchronize()
    mse = {k: v.cpu().numpy() / px for k, v in res.items()}
    for k, m in mse.items():
        with np.errstate(divide="ignore"):
            psnr = np.where(m > 0, 10 * np.log10(255.0 ** 2 / np.where(m > 0, m, 1)), np.inf)
        ape = 100 * abs(m.mean() - mse["dct"].mean()) / mse["dct"].mean() if mse["dct"].mean() > 0 else 0.0
        rows.append(f"{k},{r},{m.mean():.6f},{np.mean(psnr):.6f},{ape:.4f}")
txt = "\n".join(rows) + "\n"
if a.out:
    open(a.out, "w").write(txt)
print(txt)
