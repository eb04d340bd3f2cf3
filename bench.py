#!/usr/bin/env python
"""Benchmark of the B200 FBS hot path (BASELINE.json metric: Mdisp/s and fps per
stereo pair, Teddy-shaped 450x375x60, at 1/2/4/8 B200, vs roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config teddy|tsukuba|kitti|mb2014]
                  [--impl ours|reference]

One step = the whole hot path (stats -> twin costs -> aggregation + WTA both
sides -> LRC + subpixel) on one synthetic stereo pair per rank, inputs
resident in HBM.  L2 is flushed (a 256 MiB write) between timed steps, outside
the per-step CUDA events.  Under torchrun (N > 1): teddy/tsukuba/kitti shard
frames across ranks (weak scaling, no data-path collective); mb2014 splits one
frame into row bands + an NCCL all-gather (strong scaling).  Rank 0 prints ONE
JSON line.  ``--impl reference`` times the CPU oracle (the reference arm of
this tier) on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import stereo_synth as synth  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")
NOMINAL_FP32_LANES_PER_SM = 128  # B200: 4 SMSP x 32 FP32 lanes (B200_PROFILING.md: 148 SMs)
# measured register-only FFMA2 (broadcast scalar operand) throughput on this pool's B200s
# (tools/microbench/ffma_peak.cu, profiles/r01_ffma_microbench.txt): the practical ceiling
FFMA2_CEILING_TFLOPS = 66.9


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def mdisp(cfg, frames: float, seconds: float) -> float:
    """Eq.(13) P:L337-341 with the range width D = d_max - d_min + 1 (R#24)."""
    return cfg.W * cfg.H * cfg.D * frames / seconds * 1e-6


def useful_flops_per_side(cfg) -> float:
    """Numerator FMAs of Eq.(6) only: W*H*D*(2rho+1)^2 per volume, 2 flop each."""
    return 2.0 * cfg.W * cfg.H * cfg.D * (2 * cfg.radius + 1) ** 2


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock and throttle reasons
    while the timed region runs."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            h = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(device_index).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU") else uuid)
            except Exception:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                idx = int(vis.split(",")[device_index]) if vis and vis.split(",")[0].isdigit() else device_index
                h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.h = h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: record the absence
            log("clock sampler unavailable:", e)
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def cpu_baseline(cfg, frames_np, budget_s: float = 20.0) -> dict:
    """The oracle as it stands, on this host's cores, on a bounded sample."""
    import oracle
    th = os.cpu_count() or 1
    n, t = 0, 0.0
    for L, R in frames_np:
        t0 = time.perf_counter()
        oracle.fbs(L, R, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r, threads=th,
                   volumes=False)
        t += time.perf_counter() - t0
        n += 1
        if t > budget_s:
            break
    return {"value": mdisp(cfg, n, t), "unit": "Mdisp/s", "cores": th, "kind": "oracle",
            "sample": f"{n} full {cfg.name} frame(s) {cfg.W}x{cfg.H} D={cfg.D} rho={cfg.radius}, "
                      f"{th} OpenMP threads, {t:.1f} s"}


def load_peak_fp32():
    """ALU roofline denominator: 148 SMs x 128 FP32 lanes x 2 flop x max SM clock,
    the clock from MEASURED_PEAKS.json (driver-written) else the guide's 1965 MHz."""
    mhz, src = 1965.0, "B200_PROFILING.md clocks.max.sm 1965 MHz"
    try:
        mp = json.load(open(PEAKS_PATH))
        mhz, src = float(mp["sm_max_mhz"]), "MEASURED_PEAKS.json sm_max_mhz"
    except Exception:
        pass
    return 148 * NOMINAL_FP32_LANES_PER_SM * 2 * mhz * 1e6 / 1e12, src


def load_traffic(cfgname, path):
    """dram read+write bytes of one launch of the dominant kernel, from the committed
    ncu --set full summary (profiles/ncu_summary.json), else None."""
    try:
        s = json.load(open(PROFILE_SUMMARY))
        return s.get(f"{cfgname}/{path}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def bench_config(cfg, world, batch=1):
    """The `config` object of the JSON line — identical for both arms (the driver
    compares them): the workload, its partition across ranks and the inputs."""
    banded = cfg.name == "mb2014"
    return {"workload": f"{cfg.name} {cfg.W}x{cfg.H} d={cfg.d_min}..{cfg.d_max} (D={cfg.D}) "
                        f"rho={cfg.radius} gamma_d={cfg.gamma_d} gamma_r={cfg.gamma_r}",
            "frames_per_step_per_rank": batch,
            "partition": (f"row bands x{world} + NCCL all-gather" if banded else
                          f"frame sharding x{world}, no data-path collective"),
            "l2": "256 MiB L2 flush between timed steps (outside the step events)",
            "input_sha256": synth.digest(*synth.frame(cfg, 0))[:16]}


# ---------------------------------------------------------------------------
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_1807_02044_b200 as fbs
    from paper_1807_02044_b200 import dist as fdist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    banded = cfg.name == "mb2014"
    B = 1 if banded else args.batch  # frames per step (NEXT-2: fbs_compute_batch, one launch per <= 16 frames
                                     # on the fused path)
    nfr = 1 if banded else max(4, B)
    frames_np = [synth.frame(cfg, i + (0 if banded else 1000 * rank)) for i in range(nfr)]
    Ls = [torch.from_numpy(L).to(dev) for L, _ in frames_np]
    Rs = [torch.from_numpy(R).to(dev) for _, R in frames_np]
    # row bands (N > 1): each rank's handle covers only its band (fbs_create_band)
    band = fdist.band_range(cfg.H, rank, world) if banded and world > 1 else None
    m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r, path=args.path,
                rows=band if band and band[1] > band[0] else None)
    out = torch.empty((cfg.H, cfg.W), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    if B > 1:  # stacked batches, rotating through the frames
        nb = 4
        Lb = [torch.stack([Ls[(j * B + k) % nfr] for k in range(B)]) for j in range(nb)]
        Rb = [torch.stack([Rs[(j * B + k) % nfr] for k in range(B)]) for j in range(nb)]
        outb = torch.empty((B, cfg.H, cfg.W), dtype=torch.float32, device=dev)

    if args.sparse_margin is not None:  # NEXT-4: seeds = the full-range maps (a stream's previous frames)
        seeds = [m.compute(Ls[i], Rs[i]) for i in range(nfr)] if world == 1 else None
        torch.cuda.synchronize()

    def step(i):
        L, R = Ls[i % nfr], Rs[i % nfr]
        if args.sparse_margin is not None and world == 1:
            rl, rr = m.suggest_ranges(seeds[i % nfr], args.sparse_margin)
            m.compute_ranged(L, R, rl, rr, out=out)
        elif B > 1:
            m.compute_batch(Lb[i % nb], Rb[i % nb], out=outb)
        elif banded and args.band_scatter and world > 1:  # NEXT-3: peer stores into symmetric memory
            fdist.compute_banded_scatter(m, L, R, cfg.H, cfg.W, rank, world)
        elif banded:
            fdist.compute_banded(lambda r0, r1, band: m.compute_rows(L, R, r0, r1, out=band[: r1 - r0]),
                                 cfg.H, cfg.W, rank, world, device=dev)
        else:
            m.compute(L, R, out=out)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    launches = m.launches_per_frame()
    # the timed steps replay CUDA graphs of fbs_compute (one per input frame; SURVEY
    # §8(d)): fbs_compute only enqueues, so it captures as is
    graphs = []
    if not banded and not args.no_graph and args.sparse_margin is None:
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            for i in range(nfr if B == 1 else nb):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    if B == 1:
                        m.compute(Ls[i], Rs[i], out=out, stream=cs)
                    else:
                        m.compute_batch(Lb[i], Rb[i], out=outb, stream=cs)
                graphs.append(g)
        torch.cuda.synchronize()
        for i in range(args.warmup):
            graphs[i % len(graphs)].replay()
        torch.cuda.synchronize()

    def timed_step(i):
        if graphs:
            graphs[i % len(graphs)].replay()
        else:
            step(i)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    t_wall = time.perf_counter()
    with sampler:
        for i in range(args.steps):
            flush.fill_(float(i))            # untimed L2 flush (256 MiB > 126 MB L2)
            ev[i][0].record(stream)
            timed_step(i)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    # per-kernel durations: a profiled pass of the same steps right after the timed
    # region (stage events between the launches would serialise the programmatic
    # dependent launches, so they stay out of the timed steps)
    nprof_steps = min(args.steps, 500)
    m.profile_enable(nprof_steps * B)  # events per launch sequence: per frame (volume) or per batch (fused)
    for i in range(nprof_steps):
        flush.fill_(float(i))
        step(i)
    torch.cuda.synchronize()
    stage_ms, nprof = m.profile_read()
    tiles = m.tile_stats()
    m.profile_enable(0)
    t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    frames_total = args.steps * (1 if banded else world * B)
    value = mdisp(cfg, frames_total, max_ms / 1e3)

    # ---- end to end through the public C ABI with pinned host buffers ----
    e2e = None
    if not banded and not args.no_extras:
        # a step = one pipelined batch of EB frames from pinned host memory through
        # fbs_compute_host_batch (uploads / downloads overlap the compute of
        # neighbouring frames); L2 flushed between steps
        EB = args.e2e_batch
        hl = torch.from_numpy(np.stack([frames_np[i % nfr][0] for i in range(EB)])).pin_memory()
        hr = torch.from_numpy(np.stack([frames_np[i % nfr][1] for i in range(EB)])).pin_memory()
        hout = torch.empty((EB, cfg.H, cfg.W), dtype=torch.float32).pin_memory()
        ne = max(3, min(args.steps, 4000 // EB))
        for i in range(3):
            m.compute_host_batch(hl, hr, out=hout, stream=stream)
        if world > 1:
            dist.barrier()
        e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ne)]
        for i in range(ne):
            flush.fill_(float(i))
            e_ev[i][0].record(stream)
            m.compute_host_batch(hl, hr, out=hout, stream=stream)
            e_ev[i][1].record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in e_ev)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        # single-frame latency of the blocking host call (wall clock around
        # fbs_compute_host: upload, compute, download, synchronise), L2 flushed before each
        h1l, h1r = hl[0].clone().pin_memory(), hr[0].clone().pin_memory()
        h1o = torch.empty((cfg.H, cfg.W), dtype=torch.float32).pin_memory()
        lat = []
        for i in range(3 + 50):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m.compute_host(h1l, h1r, out=h1o, stream=stream)
            if i >= 3:
                lat.append(time.perf_counter() - t0)
        e2e = {"value": mdisp(cfg, ne * EB * world, float(e_ms.item()) / 1e3), "unit": "Mdisp/s",
               "h2d_bytes_per_step": 2 * cfg.W * cfg.H * EB, "d2h_bytes_per_step": 4 * cfg.W * cfg.H * EB,
               "frames_per_step": EB, "fps": ne * EB * world / (float(e_ms.item()) / 1e3),
               "api": "fbs_compute_host_batch (pinned host buffers, pipelined copies; the step's first "
                      "upload starts after the step's start event)",
               "single_frame_latency_ms": round(1e3 * statistics.median(lat), 4),
               "single_frame_api": "fbs_compute_host, one frame, blocking, wall clock (median of 50)"}

    if rank != 0:
        return None
    # ---- roofline of the dominant kernel (aggregation + WTA, both sides in one launch) ----
    peak, peak_src = load_peak_fp32()
    agg_ms = stage_ms["main"] / max(1, nprof)
    if banded:
        rows = fdist.band_range(cfg.H, rank, world)
        frac_rows = (rows[1] - rows[0]) / cfg.H
    else:
        frac_rows = 1.0
    fpe = nprof_steps * B / max(1, nprof)  # frames per profiled launch (fused batches: up to 16)
    achieved = 2 * useful_flops_per_side(cfg) * frac_rows * fpe / (agg_ms * 1e-3) / 1e12
    tot_stage = sum(stage_ms.values())
    roof = {"bound": "alu", "achieved": round(achieved, 3), "peak": round(peak, 2), "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": load_traffic(cfg.name, args.path),
            "kernel": ("k_agg (bilateral aggregation + WTA, both sides per launch; costs read from the "
                       "L2/HBM volumes k_cost wrote)" if args.path == "volume" else
                       "k_fbs_ws (fused: NCC costs into a shared-memory ring + aggregation + WTA, both sides)"),
            "avg_launch_ms": round(agg_ms, 5),
            "timing": "dominant-kernel launch duration from CUDA events on the launching stream around each "
                      "launch, in a profiled pass of the same workload right after the timed steps",
            "share_of_step": round(stage_ms["main"] / tot_stage, 3) if tot_stage else None,
            "stage_ms_per_frame": {(("cost", "agg", "finalize") if args.path == "volume" else
                                    ("prep", "fbs", "final"))[i]: round(v / max(1, nprof) / fpe, 5)
                                   for i, v in enumerate(stage_ms.values())},
            "frames_per_launch": fpe,
            "peak_source": f"148 SM x 128 FP32 lanes x 2 x {peak_src} (nominal); "
                           "FFMA2 microbenchmark 66.9 TFLOP/s (DESIGN.md §6)",
            "frac_of_ffma2_ceiling": round(achieved / FFMA2_CEILING_TFLOPS, 4),
            "l1_bound": ("volume path: 0.69 L1 data-pipe wavefronts per FFMA2 (ncu per-instruction "
                         "counts) cap k_agg at 72 % of FP32 peak before latency / prologue / tail "
                         "losses (profiles/r02_agg_lsu_budget.txt, DESIGN.md §9b)") if args.path == "volume" else None,
            "useful_work": "numerator FMAs of Eq.(6): 2 sides x W*H*D*(2rho+1)^2 per launch",
            "denominator_forms": {k: round(v / max(1, sum(tiles.values())), 4) for k, v in tiles.items()}}
    base = None
    if world == 1 and not args.no_extras:
        # about 10 s of oracle work: whole frames, cycled until the budget is spent
        base = cpu_baseline(cfg, (list(frames_np) * 200)[:200] if not banded else frames_np[:1], budget_s=10.0)
    res = {
        "metric": "Mdisp/s",
        "value": round(value, 1),
        "unit": "Mdisp/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(max_ms / args.steps, 5),
        "fps": round(frames_total / (max_ms / 1e3), 1),
        "higher_is_better": True,
        "scaling": "strong" if banded else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded layered Middlebury-like pairs, stereo_synth v%d)" % synth.SYNTH_VERSION,
        "config": bench_config(cfg, world, B),
        "path": args.path,
        "mode": (f"sparse search range (NEXT-4): per step fbs_suggest_ranges(margin={args.sparse_margin}) from "
                 "the frame's full-range map + fbs_compute_ranged" if args.sparse_margin is not None
                 else "full search range"),
        "timing": ("CUDA-graph replay of fbs_compute per step" if graphs else "eager launches per step"),
        "roofline": roof,
        "cpu_baseline": base,
        "e2e": e2e,
        "gpu_launches": launches * args.steps,
        "clocks": sampler.summary(),
        "wall_s_timed_region": round(t_wall, 4),
        "impl": "ours",
    }
    return res


def run_reference(args, cfg, rank):
    """Reference arm of this tier: the CPU oracle as it stands, on this host's
    cores.  Each step = the full method on a band of B output rows (+ its
    rho+1-row input halo, so the band's output is exact), B sized so the run
    ends within a few minutes."""
    import oracle
    if rank != 0:
        return None
    th = os.cpu_count() or 1
    L, R = synth.frame(cfg, 0)
    halo = cfg.radius + 1

    def band_step(r0, B):
        a, b = max(0, r0 - halo), min(cfg.H, r0 + B + halo)
        t0 = time.perf_counter()
        oracle.fbs(L[a:b], R[a:b], cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r,
                   threads=th, volumes=False)
        return time.perf_counter() - t0

    # size the band: ~90 s for the timed steps
    t1 = band_step(cfg.H // 2, 8) / (8 + 2 * halo)
    budget = float(os.environ.get("FBS_REF_BUDGET_S", "90"))
    B = int(max(1, min(cfg.H, budget / max(1, args.steps) / t1 - 2 * halo)))
    for i in range(args.warmup):
        band_step((i * B) % max(1, cfg.H - B), B)
    tt = 0.0
    for i in range(args.steps):
        tt += band_step((i * B) % max(1, cfg.H - B), B)
    value = cfg.W * B * cfg.D * args.steps / tt * 1e-6
    sample = (f"per step: oracle on a {B}-row band (+{halo}-row halo) of the same {cfg.name} "
              f"{cfg.W}x{cfg.H} D={cfg.D} frame (frame 0 of the config), {th} threads")
    return {"metric": "Mdisp/s", "value": round(value, 3), "unit": "Mdisp/s", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tt / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": bench_config(cfg, int(os.environ.get("WORLD_SIZE", "1"))),
            "cpu_baseline": {"value": round(value, 3), "unit": "Mdisp/s", "cores": th, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "Mdisp/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="teddy", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="volume", choices=["volume", "fused"],
                    help="implementation path (fbs_create_ex): volume (default, fastest) or fused")
    ap.add_argument("--e2e-batch", type=int, default=8,
                    help="frames per end-to-end step (fbs_compute_host_batch pipeline depth)")
    ap.add_argument("--radius", type=int, default=None,
                    help="override the config's aggregation radius rho (NEXT-1 sweep; paper's operating point is 6)")
    ap.add_argument("--batch", type=int, default=1,
                    help="frames per step through fbs_compute_batch (NEXT-2; not for mb2014)")
    ap.add_argument("--sparse-margin", type=int, default=None,
                    help="NEXT-4: per step, suggest ranges (margin M) from the frame's full-range map "
                         "and run the ranged WTA (sparse search range)")
    ap.add_argument("--band-scatter", action="store_true",
                    help="mb2014 at N > 1: bands stored into the peers' symmetric-memory buffers (NEXT-3) "
                         "instead of the NCCL all-gather")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of CUDA-graph replays")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the e2e and cpu_baseline legs (for profiler runs)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    cfg = synth.CONFIGS[args.config]
    if args.radius is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, radius=args.radius)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"note: WORLD_SIZE={world} but --gpus={args.gpus}; using WORLD_SIZE")
    if args.impl == "reference":
        res = run_reference(args, cfg, rank)
    else:
        import torch
        import torch.distributed as dist
        # FBS_BENCH_BACKEND=gloo: a dry run of the multi-rank logic (frame sharding, row
        # bands + gather, max-over-ranks timing) with more ranks than GPUs; the line is
        # marked "dry_run" and is not a measurement.  The default is NCCL, one GPU per rank.
        backend = os.environ.get("FBS_BENCH_BACKEND", "nccl")
        dev_index = local_rank
        if world > 1:
            if backend == "nccl":
                torch.cuda.set_device(local_rank)
                dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
            else:
                if args.band_scatter:
                    ap.error("--band-scatter needs NCCL and one GPU per rank")
                dev_index = local_rank % torch.cuda.device_count()
                torch.cuda.set_device(dev_index)
                dist.init_process_group(backend)
        res = run_ours(args, cfg, rank, world, dev_index)
        if res is not None and world > 1 and backend != "nccl":
            res["dry_run"] = (f"{backend} backend, {world} ranks on {torch.cuda.device_count()} GPU(s): "
                              "checks the multi-rank logic only, not a measurement")
        if world > 1:
            dist.destroy_process_group()
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
