"""One-off full-size validation (evidence for DESIGN.md, not a test): N C5 images (4096^2, the bench
generator, global indices spread over the 4096-image corpus so all three kinds appear), every r of
the bench, GPU SSE (the bench's launch configuration) against the float64 CPU oracle on the same
bytes; also the fused multi-r kernel.  Prints the max relative SSE difference and max |dPSNR|.

    python tools/validate_c5.py [N] > profiles/r01_c5_validation.txt
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1402_6034_b200 as A  # noqa: E402
from synth import images as S  # noqa: E402

RS = (1, 3, 6, 10, 15, 21, 28, 36)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    idx = [int(i) for i in np.linspace(0, 4095, n)]
    worst_rel, worst_db, worst_multi = 0.0, 0.0, 0.0
    t0 = time.time()
    for gi in idx:
        x = S.device_mixed(1, 4096, 4096, seed=0, device="cuda", first_index=gi)
        gpu = np.stack([A.compress_psnr(x, r).cpu().numpy()[0] for r in RS])
        multi = A.compress_psnr_multi(x, RS).cpu().numpy()[:, 0]
        img = x.cpu().numpy()
        want = np.stack([O.compress_zonal_sse(img, r)[0] for r in RS])
        rel = np.abs(gpu - want) / np.maximum(want, 1e-6 * 4096 * 4096)
        db = np.abs(O.psnr(gpu, 4096 * 4096) - O.psnr(want, 4096 * 4096))
        worst_rel, worst_db = max(worst_rel, rel.max()), max(worst_db, db.max())
        worst_multi = max(worst_multi, (np.abs(multi - gpu) / np.maximum(gpu, 1e-30)).max())
        print(f"image {gi:4d} (kind {gi % 3}): max rel SSE diff {rel.max():.2e}, max |dPSNR| {db.max():.2e} dB, "
              f"PSNR r=1..36: " + " ".join(f"{v:.2f}" for v in O.psnr(want, 4096 * 4096)), flush=True)
    print(f"# {n} C5 images x {len(RS)} r vs the float64 oracle: max rel SSE diff {worst_rel:.2e} (bar 1e-5), "
          f"max |dPSNR| {worst_db:.2e} dB (bar 1e-3); fused multi-r vs single passes: {worst_multi:.2e}; "
          f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
