"""World-size-2 checks of the multi-rank path on CPU (gloo): image sharding, the SSE all-reduce and
the max-over-ranks timing reduction.  Per-shard SSE comes from the oracle (no GPU here); the test
checks that the combined buffer equals the single-process result exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1402_6034_b200.dist import combine_sse, max_over_ranks, shard_range
from synth import images as S

R_SET = (1, 3, 10, 36)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_path):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    imgs = S.corpus_c2(n, 32, 48)
    lo, hi = shard_range(n, rank, world)
    sse = torch.zeros((len(R_SET), n), dtype=torch.float64)
    for k, r in enumerate(R_SET):
        if hi > lo:
            sse[k, lo:hi] = torch.from_numpy(O.compress_zonal_sse(imgs[lo:hi], r))
    combine_sse(sse)
    t = max_over_ranks(10.0 + rank)
    if rank == 0:
        np.save(out_path, sse.numpy())
        np.save(out_path + ".t.npy", np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [5, 6, 1])
def test_two_rank_sse_allreduce_matches_single_process(tmp_path, n):
    out = str(tmp_path / "sse.npy")
    mp.spawn(_worker, args=(2, _free_port(), n, out), nprocs=2, join=True)
    got = np.load(out)
    imgs = S.corpus_c2(n, 32, 48)
    want = np.stack([O.compress_zonal_sse(imgs, r) for r in R_SET])
    assert np.array_equal(got, want)
    assert np.load(out + ".t.npy")[0] == 11.0


def test_shard_range_partitions():
    for n in (0, 1, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
