"""bench.py -- the driver's benchmark contract for the abin hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1|2|3|4|5|5b] [--scaling strong|weak]

One step = one pass of the whole hot path (moments -> Sauvola threshold ->
mask) over one batch of synthetic pages resident in HBM.  The default
workload is BASELINE.json config 3 (the large-page config the >= 70 % roofline
target is quoted on): a batch of 64 pages of 7016 x 4960 uint8 (A4 @ 600 dpi)
with the stain blob, Sauvola k = 0.5, R = 128, h = w = 61, byte mask.  Pages
are independent: at N GPUs the 64-page batch is sharded 64/N pages per rank
(strong scaling, BASELINE configs[2]; no data-path collective); --scaling weak
gives every rank its own 64 pages instead.  --config 5b is BASELINE configs[4]'s
page batch: 32 pages of 4096^2, local median 51x51, sharded over the ranks.
--config 2 times the window sweep h = w in {15, 31, 63, 127, 255} (one step =
the five windows) and reports each window and the flatness (max / median).
--config 4 at N > 1 splits the 32768^2 scan into row bands with NCCL halos.
Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, the only other place bench.py
executes it) on the host cores, on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (input generator: no method arithmetic)

METRIC = "binarized gigapixels/s (Sauvola) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Gpx/s"

CONFIGS = {
    # cfg: (pages, H, W, h, w, method, k, R, packed, stain, label)
    1: (1, 512, 512, 32, 32, "sauvola", 0.5, 128.0, False, False,
        "config1: 1 page 512x512 u8, Sauvola k=0.5 R=128 h=w=32, u8 mask"),
    2: (1, 3300, 2550, 63, 63, "sauvola", 0.5, 128.0, False, False,
        "config2: 1 page 3300x2550 u8 (letter @300dpi), Sauvola k=0.5 R=128 h=w=63, u8 mask"),
    3: (64, 7016, 4960, 61, 61, "sauvola", 0.5, 128.0, False, True,
        "config3: 64 pages x 7016x4960 u8 (A4 @600dpi) + stain, Sauvola k=0.5 R=128 h=w=61, u8 mask"),
    4: (1, 32768, 32768, 101, 101, "sauvola", 0.34, 128.0, True, False,
        "config4: 1 page 32768x32768 u8, Sauvola k=0.34 R=128 h=w=101, forced u64 square sums, bit mask"),
    5: (1, 4096, 4096, 51, 51, "quantile", 0.5, 0.0, False, False,
        "config5: 1 page 4096x4096 u8, local median (q=0.5) 51x51, u8 mask"),
    "5b": (32, 4096, 4096, 51, 51, "quantile", 0.5, 0.0, False, False,
           "config5b: batch of 32 pages 4096x4096 u8, local median (q=0.5) 51x51, u8 mask"),
}
SWEEP = (15, 31, 63, 127, 255)  # config 2's windows (BASELINE configs[1])
SWEEP_BATCH = 16                # pages of the throughput-bound companion sweep (batched_sweep)


def cfg_key(c):
    return c if c == "5b" else int(c)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(cfg, px_per_launch):
    """dram read+write bytes per launch of the dominant kernel, from the
    committed `ncu --set full` summary (profiles/ncu_summary.json, written by
    tools/summarize_profile.py); None unless it was captured on this config
    with the same launch size."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    e = json.load(open(path)).get(f"config{cfg}")
    if e is None or int(e.get("px_per_launch", -1)) != int(px_per_launch):
        return None
    return e.get("dram_bytes_per_launch")


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, torch_dev):
        self.samples, self.reasons, self.ok = [], 0, False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            h = None
            try:  # match the CUDA device to its NVML handle by UUID
                import torch
                want = str(torch.cuda.get_device_properties(torch_dev).uuid).lower()
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hi = pynvml.nvmlDeviceGetHandleByIndex(i)
                    u = pynvml.nvmlDeviceGetUUID(hi)
                    u = (u.decode() if isinstance(u, bytes) else u).lower()
                    if want and want in u:
                        h = hi
                        break
            except Exception:
                h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(torch_dev.index or 0)
            self.h = h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # NVML missing: report nothing rather than guess
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [k for k, v in self.REASONS.items() if self.reasons & v]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------- distributed

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def page_shard(P, rank, world, scaling):
    """(first page, pages) of this rank: the batch sharded contiguously and
    balanced (strong scaling), or a whole batch per rank (weak)."""
    if scaling == "weak" or world == 1:
        return rank * P, P
    base, extra = divmod(P, world)
    return rank * base + min(rank, extra), base + (1 if rank < extra else 0)


def make_pages(cfg, rank, scaling, world):
    P, H, W, h, w, method, k, R, packed, stain, _ = CONFIGS[cfg]
    first, n = page_shard(P, rank, world, scaling)
    pages = np.empty((n, H, W), np.uint8)
    seed_cfg = 5 if cfg == "5b" else cfg
    if n:
        synth.pages(n, H, W, synth.config_seed(seed_cfg, first), stain=stain, out=pages)
    return pages


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference_main(args):
    """--impl reference: the CPU oracle as it stands, rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    cfg = args.config
    P, H, W, h, w, method, k, R, packed, stain, label = CONFIGS[cfg]
    page = np.empty((H, W), np.uint8)
    synth.page(H, W, synth.config_seed(5 if cfg == "5b" else cfg, 0), stain=stain, out=page)
    cores = oracle.num_threads()
    # bounded sample: a full-width band of rows of page 0, sized (from a
    # calibration band) so the whole warm-up + timed run takes ~2 minutes
    per_step = min(3.0, max(0.2, 120.0 / max(1, args.steps + args.warmup)))
    rows = min(H, 4)
    t0 = time.perf_counter()
    _oracle_band(oracle, method, page, rows, h, w, k, R)
    dt = max(time.perf_counter() - t0, 1e-6)
    rows = int(max(1, min(H, rows * per_step / dt)))
    for _ in range(args.warmup):
        _oracle_band(oracle, method, page, rows, h, w, k, R)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _oracle_band(oracle, method, page, rows, h, w, k, R)
        times.append(time.perf_counter() - t0)
    px = rows * W
    tmean = sum(times) / len(times)
    value = px / tmean / 1e9
    sample = f"rows 0..{rows - 1} (full width {W}) of page 0 of {label}; {px} px per step"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tmean * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg in (3, "5b", 4) and args.scaling == "strong" else "weak",
            "vs_baseline": None, "dtype": "u64/f64", "data": "synthetic",
            "config": {"workload": label, "sample_rows": rows},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _oracle_band(oracle, method, page, rows, h, w, k, R):
    """Oracle on output rows [0, rows) of `page` (full width): the oracle sees
    the rows the windows need and the page's true height for n."""
    H, W = page.shape
    rr = np.repeat(np.arange(rows, dtype=np.int64), W)
    cc = np.tile(np.arange(W, dtype=np.int64), rows)
    if method == "quantile":
        return oracle.quantile_points(page, h, w, k, rr, cc)
    return oracle.binarize_points(method, page, h, w, k, R, -1, rr, cc)


def cpu_baseline(cfg, budget_s=12.0):
    """The oracle, as it stands, on a bounded sample of the workload."""
    import oracle
    P, H, W, h, w, method, k, R, packed, stain, label = CONFIGS[cfg]
    page = np.empty((H, W), np.uint8)
    synth.page(H, W, synth.config_seed(5 if cfg == "5b" else cfg, 0), stain=stain, out=page)
    rows = min(H, 4)
    t0 = time.perf_counter()
    _oracle_band(oracle, method, page, rows, h, w, k, R)
    dt = max(time.perf_counter() - t0, 1e-6)
    rows2 = int(max(1, min(H, rows * (budget_s * 0.8) / dt)))
    t0 = time.perf_counter()
    _oracle_band(oracle, method, page, rows2, h, w, k, R)
    dt2 = time.perf_counter() - t0
    px = rows2 * W
    return {"value": px / dt2 / 1e9, "unit": UNIT, "cores": oracle.num_threads(), "cpu_model": cpu_model(),
            "kind": "oracle",
            "sample": f"direct definition on rows 0..{rows2 - 1} (full width) of page 0 of {label}: "
                      f"{px} px in {dt2:.2f} s"}


L2_BYTES = 126e6


def batched_sweep(ab, page, k, R, dev, stream, n_pages=SWEEP_BATCH, reps=5):
    """Config 2's windows on a batch of n_pages copies of the letter page (one
    binarize_batched launch per window, CUDA events on the launching stream).
    A single 3300x2550 page keeps only part of the 148 SMs busy for tens of
    microseconds, so its sweep measures tile latency (h warm-up rows per band);
    the batch fills the device and shows the per-pixel cost against h, w --
    the paper's window-independence claim.  Inputs
    (n_pages x 8.4 MB per copy, two copies) exceed L2."""
    import torch
    H, W = page.shape
    pitch = (W + 15) // 16 * 16
    xb = torch.zeros((2, n_pages, H, pitch), dtype=torch.uint8, device=dev)
    xb[:, :, :, :W] = torch.from_numpy(page).to(dev)
    ob = torch.empty((2, n_pages, H, W), dtype=torch.uint8, device=dev)
    rows = []
    for hw in SWEEP:
        for z in range(2):  # warm-up
            ab.binarize_batched("sauvola", xb[z, :, :, :W], hw, hw, k, R, out=ob[z])
        ms = []
        for i in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ab.binarize_batched("sauvola", xb[i % 2, :, :, :W], hw, hw, k, R, out=ob[i % 2])
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        msz = statistics.median(ms)
        rows.append({"h": hw, "w": hw, "ms": msz, "gpx_s": n_pages * H * W / msz / 1e6})
    med = statistics.median(r["gpx_s"] for r in rows)
    del xb, ob
    return {"pages": n_pages, "rows": rows,
            "flatness": {"max_over_median": max(r["gpx_s"] for r in rows) / med,
                         "min_over_median": min(r["gpx_s"] for r in rows) / med}}


def ours_main(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # ABIN_BENCH_FUNCTIONAL=1 (tests of the multi-rank code path on a box with
    # fewer GPUs than ranks): ranks share devices and talk over gloo -- a
    # functional check only, its numbers are not measurements
    functional = os.environ.get("ABIN_BENCH_FUNCTIONAL") == "1"
    if functional:
        local = local % max(1, torch.cuda.device_count())
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    import paper_1905_13038_b200 as ab
    from paper_1905_13038_b200 import abin
    from paper_1905_13038_b200 import dist as adist

    cfg = args.config
    P0, H, W, h, w, method, k, R, packed, stain, label = CONFIGS[cfg]
    sweep = cfg == 2
    if sweep:
        label = ("config2: 1 page 3300x2550 u8 (letter @300dpi), Sauvola k=0.5 R=128, window sweep h=w in "
                 + "{" + ",".join(map(str, SWEEP)) + "} (one step = the five windows), u8 mask")
    cols = (W + 7) // 8 if packed else W
    flags = abin.FORCE_U64_SQ if cfg == 4 else 0
    counters = torch.zeros(2, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    banded = cfg == 4 and world > 1
    pitch = (W + 15) // 16 * 16   # 16-byte row pitch: the TMA staging path

    if banded:
        # config 4 at N > 1: rank r owns a band of rows; halos over NCCL send/recv
        full = synth.page(H, W, synth.config_seed(cfg, 0), stain=stain)
        band = adist.make_band(H, W, h, rank, world, dev)
        band.own.copy_(torch.from_numpy(full[band.r0:band.r1]).to(dev))
        host_own = torch.from_numpy(np.ascontiguousarray(full[band.r0:band.r1])).pin_memory()
        del full
        rows = band.r1 - band.r0
        out = torch.empty((rows, cols), dtype=torch.uint8, device=dev)
        px_rank = rows * W
        n_copies = 1

        def step(i):
            adist.run_band(method, band, h, w, k, R, packed=packed, out=out, flags=flags, counters=counters,
                           rank=rank, world=world)
        # per binarize_band call: the v4 moments kernel, the exact fixup and the
        # (normally empty) v3 overflow follow-up; three calls per band
        launches_per_step = 3 * 3
        l2_note = f"band of {rows} rows per rank ({px_rank / 1e9:.2f} GB) > L2: no flush needed"
        pages_np = None
    else:
        pages_np = make_pages(cfg, rank, args.scaling, world)
        P = pages_np.shape[0]
        step_bytes = max(1, P) * H * W * (1 + cols / W)
        # inputs larger than L2: rotate through enough copies that a step never
        # finds its page (or its mask) in the 126 MB L2
        n_copies = 1 if step_bytes > 4 * L2_BYTES else int(min(2048, -(-3 * L2_BYTES // step_bytes)))
        xbuf = torch.zeros((n_copies, P, H, pitch), dtype=torch.uint8, device=dev)
        xbuf[:, :, :, :W] = torch.from_numpy(pages_np).to(dev).unsqueeze(0)
        xs = xbuf[:, :, :, :W]
        outs = torch.empty((n_copies, P, H, cols), dtype=torch.uint8, device=dev)
        out = outs[0]
        px_rank = P * H * W

        sweep_ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in SWEEP] for _ in range(args.steps + args.warmup)] if sweep else None

        # per-copy views made once (tensor indexing costs microseconds of host
        # time per step, which the short single-page steps would otherwise measure)
        views = [(xs[z], outs[z], xs[z][0] if P else None, outs[z][0] if P else None) for z in range(n_copies)]

        def step(i):
            if P == 0:
                return
            x, o, x0, o0 = views[i % n_copies]
            if sweep:
                for z, hw in enumerate(SWEEP):
                    sweep_ev[i][z][0].record(stream)
                    ab.sauvola(x0, hw, hw, k, R, packed=packed, out=o0, flags=flags, counters=counters)
                    sweep_ev[i][z][1].record(stream)
            elif P == 1:
                if method == "quantile":
                    ab.quantile(x0, h, w, k, packed=packed, out=o0)
                else:
                    ab.sauvola(x0, h, w, k, R, packed=packed, out=o0, flags=flags, counters=counters)
            else:
                ab.binarize_batched(method, x, h, w, k, R, packed=packed, out=o, flags=flags, counters=counters)
        # quantile: the v5 kernel + its exact queue (q >= 0.25; the round-1
        # kernel alone below); moments: the v5 kernel + exact fixup (+ the v3
        # overflow follow-up when the queue could overflow: its CTAs exit at
        # once unless it did); Wolf adds the fill + global-minimum pre-pass
        if method == "quantile":
            launches_per_step = 0 if P == 0 else (2 if k >= 0.25 else 1)
        else:
            launches_per_step = 0 if P == 0 else (5 if method == "wolf" else 3)
        if method != "quantile" and not sweep and not flags and P * H * W <= (1 << 22) and max(h, w) <= 64:
            # single small pages take the one-launch tile kernel (csrc/small.cuh:
            # decision inline, no fixup launch); Wolf adds the minimum pre-pass
            launches_per_step = 0 if P == 0 else (4 if method == "wolf" else 1)
        if sweep:
            launches_per_step = 3 * len(SWEEP)
        l2_note = (f"inputs {step_bytes / 1e9:.2f} GB per rank per step > L2: no flush needed" if n_copies == 1 else
                   f"L2-resident workload: steps rotate through {n_copies} input/mask copies "
                   f"({n_copies * step_bytes / 1e6:.0f} MB > 126 MB L2), no step reuses a cached page")

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    counters.zero_()

    # --- timed region (device-timed with CUDA events on the launching stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step(args.warmup + i)
            ev[i][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())

    px_step = px_rank * (len(SWEEP) if sweep else 1)
    pt = torch.tensor([float(px_step)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(pt, op=dist.ReduceOp.SUM)
    px_total = float(pt.item())          # pixels of all ranks per step
    value = px_total * args.steps / (max_ms / 1e3) / 1e9
    ms_per_step = max_ms / args.steps
    sweep_rows = None
    if sweep:
        sweep_rows = []
        for z, hw in enumerate(SWEEP):
            ms = [sweep_ev[args.warmup + i][z][0].elapsed_time(sweep_ev[args.warmup + i][z][1])
                  for i in range(args.steps)]
            msz = statistics.median(ms)
            sweep_rows.append({"h": hw, "w": hw, "ms": msz, "gpx_s": px_rank / msz / 1e6})
        sweep_batched = batched_sweep(ab, pages_np[0], k, R, dev, stream)
    auto_u32 = None
    if cfg == 4 and not banded:
        # the same page without forcing uint64: 255^2 h w < 2^32 at 101 x 101, so
        # the north star's own rule keeps uint32 square sums (the v5 kernel);
        # masks are identical (exact sums either way) -- reported beside the value
        x0, o0 = views[0][2], views[0][3]
        ab.sauvola(x0, h, w, k, R, packed=packed, out=o0)
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(stream)
        for _ in range(3):
            ab.sauvola(x0, h, w, k, R, packed=packed, out=o0)
        b_ev.record(stream)
        torch.cuda.synchronize()
        auto_u32 = {"gpx_s": 3 * px_rank / a_ev.elapsed_time(b_ev) / 1e6,
                    "note": "flags=0: uint32 square sums (255^2 h w < 2^32), v5 kernel; same mask"}

    # --- roofline of the dominant kernel: algorithmic bytes / launch time
    bytes_per_px = 1.0 + (0.125 if packed else 1.0)
    avg_kern_s = (sum(kern_ms) / len(kern_ms)) / 1e3
    achieved = px_step * bytes_per_px / avg_kern_s / 1e9
    peak, peak_kind = measured_peaks()
    traffic = None if banded else ncu_traffic(cfg, px_rank)

    # --- e2e: the same metric through the public API with HOST buffers
    # (pinned), host->device copy of the inputs and device->host copy of the
    # masks inside the timed region.
    e2e = None
    if not args.no_e2e:
        cs = torch.cuda.current_stream(dev)
        if banded:
            hout = torch.empty((rows, cols), dtype=torch.uint8).pin_memory()

            def e2e_step():
                band.own.copy_(host_own, non_blocking=True)
                adist.run_band(method, band, h, w, k, R, packed=packed, out=out, flags=flags, rank=rank,
                               world=world)
                hout.copy_(out, non_blocking=True)
            h2d, d2h = host_own.numel(), hout.numel()
        else:
            # the rank's whole shard (the headline batch: 64 pages at N = 1, 64/N
            # per rank under strong scaling), pinned; capped at 64 pages
            Pe = min(P, 64)
            hin = torch.from_numpy(np.ascontiguousarray(pages_np[:Pe])).pin_memory()
            hout = torch.empty((Pe, H, cols), dtype=torch.uint8).pin_memory()

            def e2e_step():
                if Pe == 0:
                    return
                # abin_binarize_batched with ABIN_HOST_IO: the library streams
                # the pages through device staging, copies overlapped with compute
                rc = abin.raw().abin_binarize_batched(
                    abin.METHODS[method], abin.ctypes.c_void_p(hin.data_ptr()), hin.stride(0),
                    abin.ctypes.c_void_p(hout.data_ptr()), hout.stride(0), Pe, H, W, hin.stride(1), hout.stride(1),
                    abin.MASK_BITS if packed else abin.MASK_U8, h, w, k, R, -1, flags | abin.HOST_IO, None,
                    abin.ctypes.c_void_p(cs.cuda_stream))
                if rc != 0:
                    raise abin.AbinError(rc)
            h2d, d2h = hin.numel(), hout.numel()

        e2e_steps = max(2, min(args.steps, 5))
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(cs)
        for _ in range(e2e_steps):
            e2e_step()
        b_ev.record(cs)
        torch.cuda.synchronize()
        et = torch.tensor([a_ev.elapsed_time(b_ev)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_ms = float(et.item()) / e2e_steps
        pe = torch.tensor([float(hout.shape[0] * H * W if not banded else px_rank)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(pe, op=dist.ReduceOp.SUM)
        e2e_px = float(pe.item())
        ok = torch.equal(hout, out.cpu() if banded else out[:hout.shape[0]].cpu())
        e2e = {"value": e2e_px / (e2e_ms / 1e3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms, "steps": e2e_steps,
               "pages_per_rank": None if banded else int(hout.shape[0]),
               "matches_device_path": bool(ok)}

    graph_replay = None
    if cfg == 1 and world == 1 and not banded and P == 1:
        # config 1's call is launch-bound from Python (the host spends longer per
        # call than the device): the same calls captured once in a CUDA graph and
        # replayed give the device time per call (reported beside `value`, which
        # stays the plain back-to-back calls)
        try:
            ng, reps = 200, 5
            cur = torch.cuda.current_stream()
            side = torch.cuda.Stream()
            side.wait_stream(cur)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    for i in range(ng):
                        step(i)
            cur.wait_stream(side)
            g.replay()
            torch.cuda.synchronize()
            ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ga.record(cur)
            for _ in range(reps):
                g.replay()
            gb.record(cur)
            torch.cuda.synchronize()
            us = ga.elapsed_time(gb) * 1e3 / (ng * reps)
            graph_replay = {"us_per_call": us, "gpx_s": H * W / us / 1e3, "calls_per_graph": ng, "replays": reps}
        except Exception as e:  # noqa: BLE001 -- reported, never fatal for the bench line
            graph_replay = {"error": str(e)[:200]}

    if rank == 0:
        cfgd = {"workload": label, "H": H, "W": W, "h": h, "w": w, "method": method, "k": k, "R": R,
                "mask": "bits" if packed else "u8", "l2": l2_note}
        if sweep:
            med = statistics.median(r["gpx_s"] for r in sweep_rows)
            cfgd.update(h="sweep", w="sweep", window_sweep=sweep_rows,
                        flatness={"max_over_median": max(r["gpx_s"] for r in sweep_rows) / med,
                                  "min_over_median": min(r["gpx_s"] for r in sweep_rows) / med,
                                  "criterion": "within +-20% of the median (SPEC.md:457)"},
                        window_sweep_batched=sweep_batched)
        if auto_u32 is not None:
            cfgd.update(auto_u32=auto_u32)
        if graph_replay is not None:
            cfgd.update(graph_replay=graph_replay)
        if banded:
            cfgd.update(decomposition=f"{world} row bands, halo {h // 2} rows below / {(h + 1) // 2 - 1} above "
                                      "via NCCL send/recv", rows_per_rank=px_rank // W)
        else:
            strong = args.scaling == "strong" and P0 > 1
            cfgd.update(pages_per_rank=P, batch_pages=P0 if strong else P0 * world,
                        decomposition=(f"batch of {P0} pages sharded {P0}/{world} per rank" if strong else
                                       ("every rank its own batch" if P0 > 1 else "one page per rank (replicas)"))
                        + " (no data-path collective)")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if banded or (args.scaling == "strong" and P0 > 1) else "weak",
            "vs_baseline": None, "dtype": "u32/f64",
            "data": "synthetic", "config": cfgd,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_kind": peak_kind, "algorithmic_bytes_per_px": bytes_per_px,
                         "kernel_ms": avg_kern_s * 1e3},
            "clocks": clk.summary(),
            "gpu_launches": launches_per_step * args.steps,
            "near_ties": int(counters[0].item()),
            "fallbacks": int(counters[1].item()),
        }
        if e2e is not None:
            line["e2e"] = e2e
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 50 for configs 3/4/5b, more for the short single-page steps so "
                         "the timed region spans tens of ms: 1000 for config 1, 100 for 2, 200 for 5)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=cfg_key, default=3, choices=list(CONFIGS))
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = {1: 1000, 2: 100, 5: 200}.get(args.config, 50) if args.impl == "ours" else 50
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return reference_main(args)
    return ours_main(args)


if __name__ == "__main__":
    sys.exit(main())
