"""Multi-rank path through the real CUDA kernels, on ONE GPU: two processes
(world size 2, gloo) each run adct_compress_psnr on their contiguous image shard on cuda:0, write
only their slots of a zero-initialised per-image SSE buffer [n_r, n], copy it to the host and
all-reduce it (the one collective of the path; NCCL over NVLink in bench.py, gloo here).  Blocks and
images are independent, and every per-image SSE is a fixed-point integer sum of per-tile
partials (adct_kernels.cuh fx_lane), so the all-reduced buffer must equal the single-process GPU
result BIT FOR BIT, whatever the sharding, and match the oracle on sampled images.
The ranks' kernels never wait on one another (no cross-rank device synchronisation)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle as O  # noqa: E402
from synth import images as S  # noqa: E402

R_SET = (1, 3, 6, 10, 15, 21, 28, 36)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _corpus(n, h, w):
    return S.corpus_c2(n, h, w)


def _worker(rank, world, port, n, h, w, out_path):
    import paper_1402_6034_b200 as A
    from paper_1402_6034_b200.dist import combine_sse, shard_range
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    imgs = _corpus(n, h, w)
    lo, hi = shard_range(n, rank, world)
    sse = torch.zeros((len(R_SET) + 1, n), dtype=torch.float64, device="cuda")
    if hi > lo:
        x = A.to_device(imgs[lo:hi])
        for k, r in enumerate(R_SET):
            A.compress_psnr(x, r, sse=sse[k, lo:hi])
        A.compress_psnr(x, 64, q=16.0, sse=sse[len(R_SET), lo:hi])   # C4's quantiser, frames sharded
    host_sse = sse.cpu()                       # gloo reduces host tensors
    combine_sse(host_sse)
    if rank == 0:
        np.save(out_path, host_sse.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,h,w", [(7, 256, 264), (6, 512, 512), (3, 4096, 4096)])
def test_two_ranks_cuda_shards_allreduce_bit_exact(tmp_path, n, h, w):
    import paper_1402_6034_b200 as A
    out = str(tmp_path / "sse.npy")
    mp.spawn(_worker, args=(2, _free_port(), n, h, w, out), nprocs=2, join=True)
    got = np.load(out)
    imgs = _corpus(n, h, w)
    x = A.to_device(imgs)
    single = np.stack([A.compress_psnr(x, r).cpu().numpy() for r in R_SET] +
                      [A.compress_psnr(x, 64, q=16.0).cpu().numpy()])
    assert np.array_equal(got, single)          # sharding-invariant, bit for bit
    from test_gpu_parity import check_sse
    sample = [0, n - 1]
    for k, r in enumerate(R_SET):
        check_sse(got[k, sample], O.compress_zonal_sse(imgs[sample], r), h * w)
    check_sse(got[len(R_SET), sample], O.compress_quant_sse(imgs[sample], 16.0), h * w)
