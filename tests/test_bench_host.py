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


def test_committed_bench_line_keeps_the_contract():
    """The last committed bench line (profiles/) carries every key of the bench contract."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    line = json.loads(open(os.path.join(root, "profiles", "r01_bench_N1_session4_final.jsonl")).read())
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["metric"] == json.load(open(os.path.join(root, "BASELINE.json")))["metric"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in line["roofline"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in line["cpu_baseline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in line["e2e"], k
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in line["clocks"], k
    assert line["warmup"] >= 3 and line["gpu_launches"] > 0 and line["config"]["workload"].startswith("C5")
    assert abs(line["roofline"]["frac"] - line["roofline"]["achieved"] / line["roofline"]["peak"]) < 1e-9
