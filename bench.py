"""Benchmark of the arXiv 1402.6034 hot path on B200 (BASELINE.json metric / config C5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {adct,reference}]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

Workload (BASELINE.json configs[4], "C5", the large-batch configuration the metric's HBM-roofline
target is quoted on; it fits one GPU): 4096 uint8 4096x4096 images (64 GiB) of mixed generator
kinds, zonal compression for r in {1, 3, 6, 10, 15, 21, 28, 36}: per r, forward + zonal mask +
inverse + per-image SSE (adct_compress_psnr), then an NCCL all-reduce of the per-image SSE
[8 x 4096] (N > 1) and the PSNR epilogue (adct_psnr).  The fixed C5 corpus is sharded across the
ranks (strong scaling, BASELINE C5 "Sharded 1/2/4/8"): rank k owns the contiguous image range
shard_range(4096, k, N), generated on its own GPU.  One step = all 8 r-passes over the corpus.
`--scaling weak` keeps a full 4096-image corpus per rank instead (per-GPU work fixed).
Secondary line `quant_c4`: BASELINE C4's 240 frames sharded 240/N the same way (q = 16 quantiser,
per-frame SSE all-reduced, PSNR).

Prints ONE JSON line (rank 0).  `value` = total pixel-passes / max-over-ranks device time, in
Gpixel/s; `e2e` = the same metric through adct_compress_psnr_host (pinned host images, H2D copy
+ 8 r-passes + PSNR + D2H inside the timed region) on a bounded image subset per rank;
`roofline` = the compress kernel's algorithmic 1 B/px read over its measured average launch
time vs the measured copy bandwidth in MEASURED_PEAKS.json; `cpu_baseline` = the CPU oracle
(oracle/, float64 numpy) on a bounded sample — one image per worker of a process pool over the host
cores (up to 16), plus a single-core figure — rank 0 only, N = 1 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

R_SET = (1, 3, 6, 10, 15, 21, 28, 36)
N_IMAGES, H, W = 4096, 4096, 4096
METRIC = "Gpixel/s fwd+zonal+inv+PSNR (and fwd-only) vs oracle; % of HBM roofline"
UNIT = "Gpixel/s"
WORKLOAD = "C5: 4096 x 4096x4096 uint8 (64 GiB), mixed kinds, zonal r in {1,3,6,10,15,21,28,36}"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["adct", "reference"], default="adct")
    ap.add_argument("--images", type=int, default=N_IMAGES,
                    help="corpus size (default: C5's 4096 images = 64 GiB), sharded across ranks")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the corpus is split across ranks (BASELINE C5); weak: every rank gets --images")
    ap.add_argument("--e2e-images", type=int, default=64, help="images per rank in the e2e run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fwd-only", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args()


def O_psnr(sse, pixels):
    """PSNR of host SSE values (report-only formatting of device results)."""
    import numpy as np
    sse = np.asarray(sse, dtype=np.float64)
    with np.errstate(divide="ignore"):
        return np.where(sse == 0, np.inf, 10.0 * np.log10(65025.0 * pixels / np.where(sse == 0, 1, sse)))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def committed_traffic():
    """DRAM bytes per pixel of the compress kernel from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


def issue_roofline(tr, per_r_ms, tiles_per_launch, sm_mhz, dev):
    """The compress pass is compute-bound: warp-instructions issued per second (the
    committed ncu per-tile instruction count of each r's kernel x tiles / measured launch time)
    against the issue peak of 1 warp-instruction per clock per SM sub-partition at the SM clock
    sampled during the timed region.  The ALU and FMA pipes each retire 0.5 per clock."""
    if not tr or not sm_mhz:
        return None
    import torch
    per = {}
    for name, v in tr.get("per_kernel", {}).items():
        if "k_compress<" in name and "warp_instr_per_tile" in v:
            per[int(name.split("k_compress<")[1].split(",")[0])] = v["warp_instr_per_tile"]
    if not all(r in per for r in R_SET):
        return None
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = sms * 4 * sm_mhz * 1e6  # warp-instructions per second
    ach = [per[r] * tiles_per_launch / (t * 1e-3) for r, t in zip(R_SET, per_r_ms)]
    tot = sum(per[r] * tiles_per_launch for r in R_SET) / (sum(per_r_ms) * 1e-3)
    return {"bound": "issue", "achieved": tot, "peak": peak, "unit": "warp-instr/s", "frac": tot / peak,
            "per_r_frac": {str(r): a / peak for r, a in zip(R_SET, ach)},
            "instr_source": "profiles/ncu_traffic.json warp_instr_per_tile (ncu --set full)",
            "note": "compute roofline of the same kernel: 1 warp-instr/clk/SMSP at the sampled SM clock"}


def regread_roofline(per_r_ms, tiles_per_launch, sm_mhz, dev, quant_ms=None, quant_tiles=None):
    """The binding compute resource of the fused compress kernels: register-file read
    cycles.  Achieved = the static read cycles per tile of each r's kernel (profiles/r02_regread.json,
    tools/sass_regread.py on the built objects) x tiles / measured launch time; peak = 1 read cycle per
    clock per SM sub-partition (148 x 4) at the SM clock sampled in the timed region."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_regread.json")) as f:
            rr = json.load(f)
    except Exception:
        return None
    if not sm_mhz or not all(str(r) in rr["zonal"] for r in R_SET):
        return None
    import torch
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = sms * 4 * sm_mhz * 1e6
    cyc = [rr["zonal"][str(r)]["read_cycles"] for r in R_SET]
    per = {str(r): c * tiles_per_launch / (t * 1e-3) / peak for r, c, t in zip(R_SET, cyc, per_r_ms)}
    tot = sum(c * tiles_per_launch for c in cyc) / (sum(per_r_ms) * 1e-3)
    out = {"bound": "register-file reads", "achieved": tot, "peak": peak, "unit": "read-cycles/s", "frac": tot / peak,
           "per_r_frac": per,
           # the HBM fraction each r could reach at 100 % of the read bound: (tiles / s at one read
           # cycle per clock per SMSP) / (tiles / s at the measured HBM bandwidth, 4 KiB per tile)
           "model_bound_of_hbm": {str(r): (peak / c) / (measured_peaks()[0] * 1e9 / 4096) for r, c in zip(R_SET, cyc)},
           "source": "profiles/r02_regread.json (tools/sass_regread.py); microbench evidence profiles/r02_regbank_microbench.txt"}
    if quant_ms and quant_tiles and rr.get("quant64"):
        out["quant_c4_frac"] = rr["quant64"]["read_cycles"] * quant_tiles / (quant_ms * 1e-3) / peak
    return out


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.power = []
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self.stop_ev.wait(0.05)

    def __enter__(self):
        if self.nv:
            self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.nv:
            self.th.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        out = {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
               "samples": len(self.samples)}
        if self.power:  # board power (W): the compute-bound passes run at the power-capped clock
            out["power_w_median"] = statistics.median(self.power)
        return out


def _oracle_image_task(args):
    """Pool worker: one C5 image (generated untimed) through the oracle at all 8 r.
    Returns (pixels, t_start, t_end) in host wall-clock seconds."""
    seed, kind, h, w = args
    import oracle as O
    from synth import images as S
    img = S.image_kind(seed, kind, h, w, rect_scale=8)[None]
    t0 = time.time()
    for r in R_SET:
        O.compress_zonal_sse(img, r)
    return len(R_SET) * h * w, t0, time.time()


def oracle_pool(workers: int):
    """Process pool (spawn: no CUDA state is inherited) running the oracle, one image per worker."""
    import multiprocessing as mp
    return mp.get_context("spawn").Pool(workers)


def oracle_pool_step(pool, workers: int, seed: int, h: int = H, w: int = W):
    """One parallel round: `workers` C5 images x 8 r, one per worker; throughput over the span from
    the first worker's start to the last worker's end (generation excluded, stagger included)."""
    res = pool.map(_oracle_image_task, [(seed * 7 + k, k % 3, h, w) for k in range(workers)], chunksize=1)
    px = sum(r[0] for r in res)
    wall = max(r[2] for r in res) - min(r[1] for r in res)
    return px, wall


def pool_workers() -> int:
    # bounded: each worker holds one 4096^2 image and the oracle's float64 intermediates (~1 GB)
    return max(1, min(os.cpu_count() or 1, 16))


def cpu_oracle_sample(seed: int, budget_s: float = 12.0):
    """The oracle (float64 numpy, as it stands) on C5 images, all 8 r: one parallel round over the
    host cores (process pool, one image per worker) plus a single-core run of ~budget_s / 2."""
    import oracle as O
    from synth import images as S
    workers = pool_workers()
    with oracle_pool(workers) as pool:  # worker start-up and image generation are outside the span
        ppx, pwall = oracle_pool_step(pool, workers, seed)
    imgs = [S.image_kind(seed * 7 + k, k, H, W, rect_scale=8)[None] for k in range(3)]  # untimed
    px, n_img, t_cpu0, t0 = 0, 0, os.times(), time.perf_counter()
    while time.perf_counter() - t0 < budget_s / 2 or n_img < 1:
        for r in R_SET:
            O.compress_zonal_sse(imgs[n_img % 3], r)
            px += H * W
        n_img += 1
    wall = time.perf_counter() - t0
    t_cpu1 = os.times()
    cores = max(1, round(((t_cpu1.user - t_cpu0.user) + (t_cpu1.system - t_cpu0.system)) / wall))
    return {"value": ppx / pwall / 1e9, "unit": UNIT, "cores": workers, "kind": "oracle",
            "sample": f"{workers} C5 images 4096x4096 (kinds 0..2) x 8 r, one per worker process "
                      f"(spawn pool of {workers} of {os.cpu_count()} host cores), oracle float64 numpy, "
                      f"{pwall:.1f} s span",
            "single_core": {"value": px / wall / 1e9, "cores": cores,
                            "sample": f"{n_img} C5 image(s) x 8 r in one process, {wall:.1f} s wall"}}


def run_reference(a, rank):
    """--impl reference: the CPU oracle as it stands on the box's host cores (rank 0 only): every
    step is one parallel round of one C5 image x all 8 r per worker process."""
    if rank != 0:
        return
    workers = pool_workers()
    with oracle_pool(workers) as pool:
        for i in range(a.warmup):
            oracle_pool_step(pool, workers, a.seed + 1000 + i)
        px, wall = 0, 0.0
        for i in range(a.steps):
            p_, w_ = oracle_pool_step(pool, workers, a.seed + i)
            px += p_
            wall += w_
    value = px / wall / 1e9
    sample = (f"per step {workers} C5 images 4096x4096 x 8 r, one per worker process (spawn pool of "
              f"{workers} of {os.cpu_count()} host cores), oracle float64 numpy")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": wall / a.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1402_6034_b200 as A
    from paper_1402_6034_b200.dist import combine_sse, max_over_ranks, shard_range
    from synth import images as S

    A.load()
    # functional check of the multi-rank path on a one-GPU box (NOT a measurement): every rank on
    # cuda:0 with gloo collectives (ranks never wait on each other's kernels, only on the all-reduce)
    one_dev = os.environ.get("ADCT_BENCH_ONE_DEVICE") == "1"
    local_dev = 0 if one_dev else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    n_total = a.images if a.scaling == "strong" else a.images * world
    lo, hi = shard_range(n_total, rank, world)
    n_loc = hi - lo

    # ---- inputs: this rank's shard, generated on its own GPU (untimed)
    x = S.device_mixed(n_loc, H, W, seed=a.seed, device=dev, first_index=lo)
    sse = torch.zeros((len(R_SET), n_total), dtype=torch.float64, device=dev)
    psnr = torch.empty_like(sse)
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()

    def step(evs=None):
        sse.zero_()  # other ranks' slots stay 0 for the all-reduce
        for k, r in enumerate(R_SET):
            if evs is not None:
                evs[k][0].record(stream)
            A.compress_psnr(x, r, sse=sse[k, lo:hi])
            if evs is not None:
                evs[k][1].record(stream)
        combine_sse(sse)  # the one collective: NCCL all-reduce of the per-image SSE (N > 1)
        A.psnr(sse, H * W, out=psnr)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in R_SET] for _ in range(a.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = A.launch_count()
    with ClockSampler(local_dev) as clk:
        torch.cuda.synchronize()
        t_start.record(stream)
        for s in range(a.steps):
            step(evs[s])
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = A.launch_count() - launches0
    ms = t_start.elapsed_time(t_end)
    per_r = [statistics.mean(evs[s][k][0].elapsed_time(evs[s][k][1]) for s in range(a.steps))
             for k in range(len(R_SET))]
    ms = max_over_ranks(ms, dev)
    per_r = [max_over_ranks(t, dev) for t in per_r]
    ms_step = ms / a.steps
    value = n_total * H * W * len(R_SET) / (ms_step * 1e-3) / 1e9

    # ---- parity spot check of this run's output (device result vs closed-form-free invariants)
    ps = psnr.cpu().numpy()
    assert np.all(np.isfinite(ps)) and np.all(np.diff(sse.cpu().numpy(), axis=0) <= 1e-6 * sse.cpu().numpy()[:-1] + 1e-9), \
        "SSE must be non-increasing in r"

    # ---- roofline of the dominant kernel (compress, one launch = one r-pass over the shard)
    peak, peak_src = measured_peaks()
    bytes_launch = n_loc * H * W  # algorithmic: 1 B/px read (SSE output negligible)
    avg_launch_ms = statistics.mean(per_r)
    achieved = bytes_launch / (avg_launch_ms * 1e-3) / 1e9
    tr = committed_traffic()
    traffic = None
    if tr and "dram_bytes_per_px" in tr:
        traffic = tr["dram_bytes_per_px"] * bytes_launch
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_src, "kernel": "k_compress<r,ZONAL,NONE>",
                "frac_vs_spec_8000": achieved / 8000.0,
                "per_r_frac": {str(r): bytes_launch / (t * 1e-3) / 1e9 / peak for r, t in zip(R_SET, per_r)}}
    clocks = clk.summary()
    issue = issue_roofline(tr, per_r, n_loc * (H // 16) * (W // 256), clocks.get("sm_mhz"), dev)
    regread = regread_roofline(per_r, n_loc * (H // 16) * (W // 256), clocks.get("sm_mhz"), dev)

    # ---- secondary (SURVEY F3 with the inverse, reported separately): fused multi-r kernel —
    # one read and one forward per tile, then every r's zonal step, inverse and per-pixel error
    multi_sse = torch.empty((len(R_SET), n_loc), dtype=torch.float64, device=dev)
    for _ in range(2):
        A.compress_psnr_multi(x, R_SET, sse=multi_sse)
    torch.cuda.synchronize()
    m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m0.record(stream)
    for _ in range(a.steps):
        A.compress_psnr_multi(x, R_SET, sse=multi_sse)
    m1.record(stream)
    torch.cuda.synchronize()
    mms = max_over_ranks(m0.elapsed_time(m1) / a.steps, dev)
    fused = {"what": "adct_compress_psnr_multi: one read + one forward per tile; the per-pixel errors "
                     "576x - R_r of r = 1, 3, ..., 36 by an incremental inverse (each r adds one anti-diagonal "
                     "band, exact in integers), each r's error squared pixel by pixel; NOT the headline, which "
                     "runs the 8 r-passes independently",
             "gpix_passes_s": n_total * H * W * len(R_SET) / (mms * 1e-3) / 1e9, "ms": mms,
             "speedup_vs_independent_passes": (ms_step / mms),
             "max_rel_diff_vs_independent_sse": float(((multi_sse - sse[:, lo:hi]).abs() /
                                                       sse[:, lo:hi].clamp_min(1e-30)).max().item())}
    del multi_sse

    # ---- secondary (reported separately): Parseval sweep, one read for all 8 r
    energy = torch.empty((n_loc, 16), dtype=torch.int64, device=dev)
    for _ in range(2):
        A.diag_energy(x, energy=energy, r_max=max(R_SET))
        A.sweep_psnr(energy, H * W, R_SET)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(a.steps):
        A.diag_energy(x, energy=energy, r_max=max(R_SET))
        sw_sse, _sw_psnr = A.sweep_psnr(energy, H * W, R_SET)
    s1.record(stream)
    torch.cuda.synchronize()
    sms_ = max_over_ranks(s0.elapsed_time(s1) / a.steps, dev)
    sweep = {"what": "Parseval sweep: adct_diag_energy_prefix (forward pruned to anti-diagonals 0..7 + their "
                     "exact energies + the block energy 576 sum x^2, no inverse) + adct_sweep_psnr, all 8 r "
                     "from one read; NOT the fwd+zonal+inv metric",
             "gpix_passes_s": n_total * H * W * len(R_SET) / (sms_ * 1e-3) / 1e9, "ms": sms_,
             "hbm_frac": n_loc * H * W / (sms_ * 1e-3) / 1e9 / measured_peaks()[0],
             "max_rel_diff_vs_fused_sse": float(((sw_sse[:, :] - sse[:, lo:hi]).abs() /
                                                 sse[:, lo:hi].clamp_min(1e-30)).max().item())}
    del energy

    # ---- e2e: same metric through adct_compress_psnr_host from pinned host memory
    ne = min(a.e2e_images, n_loc)
    host_imgs = torch.empty((ne, H, W), dtype=torch.uint8, pin_memory=True)
    host_imgs.copy_(x[:ne])
    dev_buf = torch.empty((ne * H * W,), dtype=torch.uint8, device=dev)
    dev_sse = torch.empty((2 * len(R_SET) * ne,), dtype=torch.float64, device=dev)
    host_psnr = torch.empty((len(R_SET), ne), dtype=torch.float64, pin_memory=True)
    del x
    copy_stream = torch.cuda.Stream()
    for _ in range(max(1, a.warmup)):
        A.compress_psnr_host(host_imgs, R_SET, dev_buf=dev_buf, dev_sse=dev_sse, host_psnr=host_psnr,
                             copy_stream=copy_stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_steps = max(3, min(a.steps, 10))
    e0.record(stream)
    for _ in range(e_steps):
        A.compress_psnr_host(host_imgs, R_SET, dev_buf=dev_buf, dev_sse=dev_sse, host_psnr=host_psnr,
                             copy_stream=copy_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ems = max_over_ranks(e0.elapsed_time(e1), dev)
    e2e = {"value": world * ne * H * W * len(R_SET) / (ems / e_steps * 1e-3) / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": ne * H * W, "d2h_bytes_per_step": len(R_SET) * ne * 8,
           "images_per_rank": ne, "api": "adct_compress_psnr_host (caller copy stream, fused multi-r kernel)",
           # the e2e step is bound by the host->device copy: its achieved PCIe rate (per rank)
           "h2d_gb_s_per_rank": ne * H * W / (ems / e_steps * 1e-3) / 1e9,
           "h2d_note": "PCIe Gen5 x16: 64 GB/s nominal per direction; the device work per copied byte "
                       "(8 r-passes) runs ~20x faster than the copy"}

    # ---- secondary (N = 1): forward-only C3 (8192 x 512^2 uniform, int16 out), 3 B/px
    fwd_only = None
    if world == 1 and not a.no_fwd_only:
        xs = S.device_uniform(8192, 512, 512, seed=a.seed, device=dev)
        out = torch.empty((8192, 512, 512), dtype=torch.int16, device=dev)
        for _ in range(3):
            A.forward(xs, out=out)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(10):
            A.forward(xs, out=out)
        f1.record(stream)
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1) / 10
        px = 8192 * 512 * 512
        fwd_only = {"workload": "C3: 8192 x 512x512 uniform u8 -> int16 Y", "gpix_s": px / (fms * 1e-3) / 1e9,
                    "ms": fms, "gb_s": 3 * px / (fms * 1e-3) / 1e9, "frac": 3 * px / (fms * 1e-3) / 1e9 / peak}
        del xs, out

    # ---- secondary: C4 quantiser (240 x 4320x7680 video frames sharded 240/N, q = 16, SSE + PSNR), 1 B/px
    quant_c4 = None
    if not a.no_fwd_only:
        nf = 240
        flo, fhi = shard_range(nf, rank, world)
        v = S.device_video(fhi - flo, 4320, 7680, seed=a.seed, device=dev, first_frame=flo)
        sse4 = torch.zeros(nf, dtype=torch.float64, device=dev)
        ps4 = torch.empty(nf, dtype=torch.float64, device=dev)

        def c4_step():
            sse4.zero_()
            if fhi > flo:
                A.compress_psnr(v, 64, q=16.0, sse=sse4[flo:fhi])
            combine_sse(sse4)
            A.psnr(sse4, 4320 * 7680, out=ps4)

        for _ in range(3):
            c4_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(5):
            c4_step()
        q1.record(stream)
        torch.cuda.synchronize()
        qms = max_over_ranks(q0.elapsed_time(q1) / 5, dev)
        px = nf * 4320 * 7680
        quant_c4 = {"workload": f"C4: 240 x 4320x7680 video frames sharded {fhi - flo}/rank over {world} GPU(s), "
                                "fwd + D-scaled quantiser q=16 + inverse + per-frame SSE all-reduce + PSNR "
                                "(k_compress<64, QUANT> residual form)",
                    "gpix_s": px / (qms * 1e-3) / 1e9, "ms": qms, "gb_s": px / (qms * 1e-3) / 1e9,
                    "frac": px / (qms * 1e-3) / 1e9 / (peak * world), "mean_psnr_db": float(ps4.mean().item())}
        del v, sse4, ps4

    # ---- secondary (N = 1): C2 sweep (45 x 512^2, r = 1..64: proposed fast path, SDCT integer fast
    # path, exact DCT dense comparator) and C1 latency (one 512^2 image, r = 10: eager and graph replay)
    c2_sweep, c1_latency = None, None
    if world == 1 and not a.no_fwd_only:
        x2 = A.to_device(S.corpus_c2())
        s2 = torch.empty((64, 45), dtype=torch.float64, device=dev)

        def r_sweep(fn):
            for r in range(1, 65):
                fn(r, s2[r - 1])

        kinds = {"proposed": lambda r, o: A.compress_psnr(x2, r, sse=o),
                 "sdct_fast": lambda r, o: A.compress_psnr_sdct(x2, r, sse=o),
                 "dct_dense": lambda r, o: A.compress_psnr_dense(x2, r, "dct", sse=o)}
        c2_sweep = {"workload": "C2: 45 x 512x512 (seeds 0..44, three kinds), r = 1..64, fwd + zonal + inv + "
                                "per-image SSE (64 launches per sweep; L2-resident, so no HBM roofline)"}
        for name, fn in kinds.items():
            r_sweep(fn)
            torch.cuda.synchronize()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            for _ in range(5):
                r_sweep(fn)
            c1.record(stream)
            torch.cuda.synchronize()
            sms2 = c0.elapsed_time(c1) / 5
            # the same 64-launch sweep captured once into a CUDA graph and replayed (the C ABI is
            # stream-ordered with host-side argument encoding only): launch gaps removed
            gs2 = torch.cuda.Stream()
            gs2.wait_stream(torch.cuda.current_stream())
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=gs2):
                for r in range(1, 65):
                    if name == "proposed":
                        A.compress_psnr(x2, r, sse=s2[r - 1], stream=gs2)
                    elif name == "sdct_fast":
                        A.compress_psnr_sdct(x2, r, sse=s2[r - 1], stream=gs2)
                    else:
                        A.compress_psnr_dense(x2, r, "dct", sse=s2[r - 1], stream=gs2)
            for _ in range(3):
                g2.replay()
            torch.cuda.synchronize()
            c0.record(stream)
            for _ in range(5):
                g2.replay()
            c1.record(stream)
            torch.cuda.synchronize()
            gms2 = c0.elapsed_time(c1) / 5
            c2_sweep[name] = {"ms_per_sweep": sms2, "gpix_passes_s": 45 * 512 * 512 * 64 / (sms2 * 1e-3) / 1e9,
                              "graph_ms_per_sweep": gms2,
                              "graph_gpix_passes_s": 45 * 512 * 512 * 64 / (gms2 * 1e-3) / 1e9,
                              "mean_psnr_db_r10": float(np.mean(O_psnr(s2[9].cpu().numpy(), 512 * 512)))}
            del g2
        x1 = A.to_device(S.image_c1(0))
        s1 = torch.empty(1, dtype=torch.float64, device=dev)
        p1 = torch.empty(1, dtype=torch.float64, device=dev)
        for _ in range(20):
            A.compress_psnr(x1, 10, sse=s1)
            A.psnr(s1, 512 * 512, out=p1)
        torch.cuda.synchronize()
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0.record(stream)
        for _ in range(200):
            A.compress_psnr(x1, 10, sse=s1)
            A.psnr(s1, 512 * 512, out=p1)
        l1.record(stream)
        torch.cuda.synchronize()
        eager_us = l0.elapsed_time(l1) / 200 * 1e3
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            A.compress_psnr(x1, 10, sse=s1, stream=gs)
            A.psnr(s1, 512 * 512, out=p1, stream=gs)
        for _ in range(20):
            g.replay()
        torch.cuda.synchronize()
        l0.record(stream)
        for _ in range(200):
            g.replay()
        l1.record(stream)
        torch.cuda.synchronize()
        c1_latency = {"workload": "C1: one 512x512 image, r = 10, compress + PSNR (3 launches)",
                      "eager_us_per_call": eager_us, "graph_replay_us_per_call": l0.elapsed_time(l1) / 200 * 1e3,
                      "psnr_db": float(p1.item())}
        del x2, s2

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_oracle_sample(a.seed)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": a.scaling,
                "vs_baseline": None, "dtype": "u8->i16x2(int32 SWAR)/f32x2", "data": "synthetic",
                "config": {"workload": WORKLOAD, "images": n_total, "images_per_gpu": n_loc, "h": H, "w": W,
                           "r": list(R_SET),
                           "parallelism": f"dp{world} ({'the fixed corpus' if a.scaling == 'strong' else 'a corpus per rank'}"
                                          f" sharded by image; one NCCL all-reduce of the per-image SSE)",
                           "l2": "inputs 64 GiB >> 126 MB L2 (no flush needed)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "issue_roofline": issue, "regread_roofline": regread, "fwd_only_c3": fwd_only, "quant_c4": quant_c4, "parseval_sweep_f3": sweep,
                "fused_multi_r_c5": fused, "c2_sweep": c2_sweep, "c1_latency": c1_latency,
                "mean_psnr_db": {str(r): float(np.mean(ps[k])) for k, r in enumerate(R_SET)}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
