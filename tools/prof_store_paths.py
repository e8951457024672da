"""Driver for an ncu capture of the TMA bulk-store paths: the C3 forward (8192 x 512^2 -> int16,
k_forward_tma<I16>), the standalone inverse int16 -> f32 / u8 (k_inverse_tma<IN, RECON>) and the zonal
compress with an f32 / u8 reconstruction (k_compress_recon), 16 x 4096^2 C5-kind images."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1402_6034_b200 as A  # noqa: E402
from synth import images as S  # noqa: E402

xs = S.device_uniform(8192, 512, 512, seed=0, device="cuda")
out = torch.empty((8192, 512, 512), dtype=torch.int16, device="cuda")
A.forward(xs, out=out)
del xs, out
x = S.device_mixed(16, 4096, 4096, seed=0, device="cuda")
y = A.forward(x)
A.inverse(y, r=64, out="f32")
A.inverse(y, r=10, out="u8")
A.compress_psnr(x, 10, recon="f32")
A.compress_psnr(x, 10, recon="u8")
torch.cuda.synchronize()
print("ok")
