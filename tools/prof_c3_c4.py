"""Driver for ncu captures of the C3 (forward-only, 8192 x 512^2 -> int16) and C4 (quantiser q = 16,
8 frames of 4320 x 7680) kernels in their own configurations."""
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
v = S.device_video(8, 4320, 7680, seed=0, device="cuda")
A.compress_psnr(v, 64, q=16.0)
torch.cuda.synchronize()
print("ok")
