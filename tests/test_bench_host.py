"""Host-side pieces of bench.py (no GPU): the oracle process pool that the cpu_baseline and the
--impl reference arm time runs the oracle unchanged, one image per worker."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import oracle as O  # noqa: E402
from synth import images as S  # noqa: E402


def test_oracle_pool_step_counts_every_pixel_pass():
    with bench.oracle_pool(2) as pool:
        px, wall = bench.oracle_pool_step(pool, 2, seed=1, h=64, w=96)
    assert px == 2 * len(bench.R_SET) * 64 * 96
    assert wall > 0


def test_oracle_image_task_runs_the_oracle_on_the_generator_image():
    px, t0, t1 = bench._oracle_image_task((5, 2, 32, 48))
    assert px == len(bench.R_SET) * 32 * 48 and t1 >= t0
    img = S.image_kind(5, 2, 32, 48, rect_scale=8)
    assert img.shape == (32, 48) and img.dtype == np.uint8
    assert np.all(np.diff([O.compress_zonal_sse(img[None], r)[0] for r in bench.R_SET]) <= 1e-7)


def test_pool_workers_bounded():
    assert 1 <= bench.pool_workers() <= 16
