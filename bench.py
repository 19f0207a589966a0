#!/usr/bin/env python
"""Benchmark driver (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload train|augment|clip|train-l14|feed]

Workloads (each has ONE metric string, `METRICS`, printed identically by both arms)
  train    (default) BASELINE.json configs[3]: ViT-B/16 fine-tune, 16x224^2 clips,
           tubelet 2x16x16 (N=1569), 64 clips per GPU; one step = K1 augmentation of
           the decoded uint8 clips + encoder fwd/bwd (tcgen05 GEMMs, blockwise
           attention) + CE loss + AdamW; data-parallel over N GPUs (NCCL all-reduce).
  augment  BASELINE.json configs[1]: K1 on 64 synthetic uint8 16x320x568 clips ->
           bf16 16x224^2 with the reference sampler's boxes.
  clip     BASELINE.json configs[2]: ViT-B/16 CLIP dual encoder, 4x224^2 clips + 77-token
           captions, 128 pairs per GPU, embedding all_gather + fused InfoNCE.
  train-l14 BASELINE.json configs[4]: ViT-L/14 16x224^2 (N=2049, D=1024, 24 layers), 24 clips/GPU.
  feed     SURVEY.md 8(f) row 1: reference-style Batch objects (host uint8 [B,16,3,224,224] ring
           views) -> DeviceFeeder (pinned ring, async H2D on a copy stream) -> K1 identity.

`--gpus N` with N > 1 re-launches itself under torch.distributed.run (N ranks, NCCL,
NCCL_DEBUG=INFO) unless it already runs under a launcher (WORLD_SIZE set).
`--impl reference` times the reference's CPU path on this host's cores, rank 0 only, with the
same metric / config / unit: libswscale for augment (the reference's scaler), the fp32
restatement (oracle/) for the training workloads.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def _baseline_metric() -> str:
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as fh:
            return json.load(fh)["metric"]
    except (OSError, ValueError, KeyError):
        return "train clips/sec ViT-B/16 16\u00d7224\u00b2 at 1/2/4/8 B200; attn TFLOP/s vs bf16 peak"


# one metric string per workload, shared by both arms so the driver can divide them
METRICS = {
    "train": _baseline_metric(),
    "train-l14": "train clips/sec ViT-L/14 16x224^2 (N=2049, 24 layers) long-sequence stress",
    "clip": "train pairs/sec ViT-B/16 CLIP dual encoder 4x224^2, InfoNCE over the global batch",
    "augment": "augment clips/sec fused RRC+flip+normalize (uint8 16x320x568 -> 16x224^2)",
    "feed": "loader->device clips/sec (host uint8 [B,16,3,224,224] -> pinned H2D -> K1 identity)",
}
UNITS = {"train": "clips/s", "train-l14": "clips/s", "clip": "pairs/s", "augment": "clips/s", "feed": "clips/s"}
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


TRAFFIC_PATH = os.path.join(ROOT, "profiles", "r02", "traffic.json")


def ncu_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed `ncu --set full` capture
    (profiles/r02/traffic.json, written by scripts/traffic_from_ncu.py), or None."""
    try:
        with open(TRAFFIC_PATH) as fh:
            ent = json.load(fh).get(kernel)
        return None if ent is None else float(ent["dram_bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        return None


def peaks() -> tuple[dict, str]:
    try:
        with open(PEAKS_PATH) as fh:
            return json.load(fh), "measured"
    except OSError:
        return dict(FALLBACK_PEAKS), "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- dist
def dist_setup(n_gpus: int):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("AVB_BENCH_SHARED_GPU") and world > 1:
        # debug only (exercises the N-rank code path on a 1-GPU box): every rank on cuda:0 over gloo;
        # the numbers are not a scaling measurement
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        return rank, world, 0
    if world > torch.cuda.device_count():
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPUs")
    if world > 1:
        # communicator lines show the N ranks; NCCL's log goes to stderr so that rank 0's stdout stays
        # exactly one JSON line (NCCL writes INFO lines to stdout unless NCCL_DEBUG_FILE is set)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    import torch

    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()


# ----------------------------------------------------------------------------- augment (config 2)
AUG_B, AUG_T, AUG_H, AUG_W = 64, 16, 320, 568


def golden_boxes(n: int) -> tuple[np.ndarray, np.ndarray]:
    path = os.path.join(ROOT, "tests", "golden", "rrc_golden.json")
    with open(path) as fh:
        g = np.asarray(json.load(fh)["config2_568x320"], dtype=np.int32)
    reps = (n + len(g) - 1) // len(g)
    g = np.concatenate([g] * reps)[:n]
    return np.ascontiguousarray(g[:, :4]), np.ascontiguousarray(g[:, 4].astype(np.uint8))


def cpu_baseline_augment(boxes, flips, budget_s: float = 12.0) -> dict:
    """The reference's CPU path (libswscale, codec.cpp:226-246) on this host's cores; falls back to
    the torch restatement when no libswscale copy loads."""
    cores = os.cpu_count() or 1
    try:
        from oracle import swscale_ref as SW

        v, n = SW.time_augment(boxes, flips, AUG_T, (AUG_H, AUG_W), budget_s, cores)
        return {"value": v, "unit": "clips/s", "cores": cores, "kind": "reference",
                "sample": f"{n} clips x {AUG_T} frames 320x568: crop -> hflip -> sws_scale(SWS_BILINEAR|"
                          f"SWS_ACCURATE_RND) to 224^2 RGB24, the reference's scaler call (codec.cpp:28-30, "
                          f"233-241) via ctypes on {SW.version_tag()}, {cores} clips in flight (GIL released); "
                          f"no normalize/cast (the reference defers them), so this flatters the CPU"}
    except RuntimeError:
        from oracle import cpu_baseline as CB

        v, n = CB.time_augment(boxes, flips, AUG_T, (AUG_H, AUG_W), budget_s, cores)
        return {"value": v, "unit": "clips/s", "cores": cores, "kind": "port",
                "sample": f"{n} clips x {AUG_T} frames 320x568 -> 224^2, torch fp32 antialiased bilinear "
                          f"restatement + normalize + bf16 cast, torch.set_num_threads({cores})"}


def workload_config(workload: str, world: int) -> dict:
    """The `config` object both arms print for a workload (weak scaling: per-GPU work fixed)."""
    if workload == "augment":
        return {"workload": "configs[1] fused GPU augmentation", "clips_per_gpu": AUG_B, "frames": AUG_T,
                "src_hw": [AUG_H, AUG_W], "target_hw": [224, 224], "global_batch": AUG_B * world,
                "parallelism": f"dp{world}", "l2": "input 558 MB > 126 MB L2 (no flush needed)"}
    if workload == "feed":
        return {"workload": "SURVEY 8(f)1 loader->device hand-off: Batch.frames uint8 [64,16,3,224,224] -> "
                            "DeviceFeeder -> K1 identity (cthw bf16)", "clips_per_gpu": FEED_B,
                "global_batch": FEED_B * world, "parallelism": f"dp{world}",
                "l2": "154 MB batch > 126 MB L2 (no flush needed)"}
    if workload == "clip":
        return {"workload": "configs[2] ViT-B/16 CLIP dual encoder 4x224^2 (N=785) + 12L/512 text, proj 256",
                "pairs_per_gpu": 128, "global_batch": 128 * world, "seq_len": 785, "parallelism": f"dp{world}",
                "l2": "per-step working set >> 126 MB L2; no flush needed"}
    large = workload == "train-l14"
    B = 24 if large else 64
    return {"workload": ("configs[4] ViT-L/14 16x224^2, tubelet 2x14x14 (N=2049), D=1024, L=24" if large else
                         "configs[3] ViT-B/16 fine-tune 16x224^2, tubelet 2x16x16 (N=1569), FlashAttention fwd/bwd"),
            "clips_per_gpu": B, "global_batch": B * world, "seq_len": 2049 if large else 1569,
            "parallelism": f"dp{world}", "optimizer": "AdamW (fused kernel)",
            "l2": "per-step working set (activations ~30 GB) >> 126 MB L2; no flush needed"}


def run_augment(args, rank, world, local):
    import torch

    from paper_2309_16669_b200 import transform as TR

    B = AUG_B
    boxes, flips = golden_boxes(B)
    g = torch.Generator(device="cuda").manual_seed(rank)
    frames = torch.randint(0, 256, (B, AUG_T, AUG_H, AUG_W, 3), generator=g, dtype=torch.uint8, device="cuda")
    boxes_d = torch.from_numpy(boxes).cuda()
    flips_d = torch.from_numpy(flips).cuda()
    out = torch.empty((B, 3, AUG_T, 224, 224), dtype=torch.bfloat16, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        TR.transform(frames, boxes_d, flips_d, out=out, crops_host=boxes)

    for _ in range(args.warmup):
        step()
    barrier(world)
    clk = ClockSampler(local)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms, world)
    value = B * world / (ms / 1e3)
    algo = TR.algorithmic_bytes(boxes, AUG_T, (224, 224), 2)
    pk, src = peaks()
    achieved = algo / (ms / 1e3) / 1e9

    # e2e: pinned host clips -> H2D -> transform -> D2H of a per-clip checksum, all timed
    host = torch.empty((B, AUG_T, AUG_H, AUG_W, 3), dtype=torch.uint8, pin_memory=True)
    host.copy_(frames.cpu())
    dev_in = torch.empty_like(frames)
    res = torch.empty((B,), dtype=torch.float32, pin_memory=True)

    def e2e_step():
        dev_in.copy_(host, non_blocking=True)
        o = TR.transform(dev_in, boxes_d, flips_d, out=out, crops_host=boxes)
        res.copy_(o.view(B, -1)[:, :1].float().view(B), non_blocking=True)

    for _ in range(2):
        e2e_step()
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)

    line = {
        "metric": METRICS["augment"],
        "value": value, "unit": "clips/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8->bf16",
        "data": "synthetic uint8 clips generated on device (torch.randint, seed=rank); boxes/flips from the "
                "reference sampler (tests/golden/rrc_golden.json)",
        "config": workload_config("augment", world),
        "roofline": {"bound": "hbm", "kernel": "k1v4_kernel", "achieved": achieved, "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": ncu_traffic("k1_rrc_normalize"),
                     "peak_source": f"{src} hbm_gbs", "algorithmic_bytes_per_launch": algo},
        "e2e": {"value": B * world / (e2e_ms / 1e3), "unit": "clips/s",
                "h2d_bytes_per_step": int(host.numel()), "d2h_bytes_per_step": int(res.numel() * 4)},
        "gpu_launches": args.steps,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_augment(boxes, flips)
    return line


# ----------------------------------------------------------------------------- feed
FEED_B, FEED_T = 64, 16


def run_feed(args, rank, world, local):
    """Reference-style Batch objects through DeviceFeeder: host ring copy + async H2D + K1 identity."""
    from dataclasses import dataclass

    import torch

    from paper_2309_16669_b200.feeder import DeviceFeeder

    @dataclass
    class Batch:               # the fields of vidpipe.loader.Batch the hand-off reads (loader.py:99-116)
        frames: np.ndarray
        sample_ids: list
        batch_index: int

    rng = np.random.default_rng(rank)
    ring = [rng.integers(0, 256, (FEED_B, FEED_T, 3, 224, 224), dtype=np.uint8) for _ in range(2)]
    feeder = DeviceFeeder(FEED_B, FEED_T, 224, 224, layout="cthw", depth=2)
    stream = torch.cuda.current_stream()
    outs = [torch.empty((FEED_B, 3, FEED_T, 224, 224), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    res = torch.empty((2,), dtype=torch.float32, pin_memory=True)

    def run(nsteps):
        batches = (Batch(ring[i % 2], list(range(FEED_B)), i) for i in range(nsteps))
        for i, out in enumerate(_feed_into(feeder, batches, outs)):
            res[i % 2:i % 2 + 1].copy_(out.view(-1)[:1].float(), non_blocking=True)   # D2H of a result

    run(args.warmup)
    torch.cuda.synchronize()
    barrier(world)
    clk = ClockSampler(local)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    e0.record(stream)
    run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = clk.stop()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)

    # device-only K1 identity (inputs resident): the roofline of the kernel behind the hand-off
    from paper_2309_16669_b200 import transform as TR

    dev = torch.from_numpy(ring[0]).cuda()
    full = np.tile(np.asarray([[0, 0, 224, 224]], np.int32), (FEED_B, 1))
    boxes_d = torch.from_numpy(full).cuda()
    for _ in range(3):
        TR.transform(dev, boxes_d, None, out=outs[0], channels_last=False, crops_host=full)
    e0.record(stream)
    for _ in range(args.steps):
        TR.transform(dev, boxes_d, None, out=outs[0], channels_last=False, crops_host=full)
    e1.record(stream)
    torch.cuda.synchronize()
    k_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    algo = FEED_B * FEED_T * 3 * 224 * 224 * 3          # uint8 read + bf16 written
    pk, src = peaks()
    ach = algo / (k_ms / 1e3) / 1e9
    value = FEED_B * world / (e2e_ms / 1e3)
    return {
        "metric": METRICS["feed"], "value": value, "unit": "clips/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": e2e_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8->bf16",
        "data": "synthetic uint8 Batch.frames (numpy, two alternating ring buffers like the reference loader)",
        "config": workload_config("feed", world),
        "roofline": {"bound": "hbm", "kernel": "k1_identity_kernel", "achieved": ach, "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": ach / pk["hbm_gbs"], "traffic": None, "peak_source": f"{src} hbm_gbs",
                     "algorithmic_bytes_per_launch": algo, "ms_per_launch": k_ms},
        "e2e": {"value": value, "unit": "clips/s", "h2d_bytes_per_step": FEED_B * FEED_T * 3 * 224 * 224 + FEED_B * 20,
                "d2h_bytes_per_step": 4, "h2d_gbs": FEED_B * FEED_T * 3 * 224 * 224 / (e2e_ms / 1e3) / 1e9},
        "note": "value is end to end (host ring copy into pinned memory + async H2D + K1 per batch, the "
                "reference's 'valid until next iter' contract); the device-only kernel rate is the roofline",
        "gpu_launches": args.steps,
        "clocks": clocks,
        **({"cpu_baseline": _feed_cpu_baseline()} if (rank == 0 and world == 1 and not args.no_cpu_baseline) else {}),
    }


def _feed_cpu_job(cores: int):
    """The reference has no device hand-off: its CPU equivalent of "uint8 Batch.frames -> normalised
    bf16 clips" is the normalise + cast it defers, restated in torch on all cores."""
    import torch

    from oracle import cpu_baseline as CB

    torch.set_num_threads(cores)
    fr = torch.randint(0, 256, (FEED_B, FEED_T, 3, 224, 224), dtype=torch.uint8)
    m = torch.tensor(CB.CLIP_MEAN).view(1, 1, 3, 1, 1)
    sd = torch.tensor(CB.CLIP_STD).view(1, 1, 3, 1, 1)

    def job():
        return ((fr.float() / 255.0 - m) / sd).permute(0, 2, 1, 3, 4).to(torch.bfloat16).contiguous()

    return job


def _feed_cpu_baseline(reps: int = 5) -> dict:
    cores = os.cpu_count() or 1
    job = _feed_cpu_job(cores)
    job()
    t0 = time.perf_counter()
    for _ in range(reps):
        job()
    sec = time.perf_counter() - t0
    return {"value": FEED_B * reps / sec, "unit": "clips/s", "cores": cores, "kind": "port",
            "sample": f"{reps} x {FEED_B} clips of uint8 [16,3,224,224] -> (x/255 - mean)/std -> bf16 [B,3,T,H,W], "
                      f"torch on {cores} host threads (the normalise + cast the reference defers, SPEC.md:232)"}


def _feed_into(feeder, batches, outs):
    """feeder.feed() with caller-owned output buffers (alternating), one batch of H2D ahead."""
    pending, k = 0, 0
    for b in batches:
        feeder.submit(b)
        pending += 1
        if pending == len(feeder.slots):
            yield feeder.next(out=outs[k % len(outs)])
            k += 1
            pending -= 1
    while pending:
        yield feeder.next(out=outs[k % len(outs)])
        k += 1
        pending -= 1


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The reference's CPU path on this host, rank 0 only; same metric / config / unit as our arm.

    Every warm-up and timed step is a real, bounded sample of the workload, and `steps` / `warmup`
    report exactly what ran; value = work done in the timed steps / their wall time."""
    if rank != 0:
        return None
    cores = os.cpu_count() or 1
    wl = args.workload
    base = {"impl": "reference", "metric": METRICS[wl], "unit": UNITS[wl], "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "config": workload_config(wl, world)}
    if wl == "feed":
        job = _feed_cpu_job(cores)

        for _ in range(args.warmup):
            job()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            job()
        sec = time.perf_counter() - t0
        v = FEED_B * args.steps / sec
        return dict(base, value=v, ms_per_step=sec / args.steps * 1e3, dtype="f32->bf16",
                    data="synthetic uint8 Batch.frames", cpu_baseline={
                        "value": v, "unit": UNITS[wl], "cores": cores, "kind": "port",
                        "sample": f"one {FEED_B}-clip batch per step: normalise + cast + re-layout in torch on "
                                  f"{cores} threads"},
                    e2e={"value": v, "unit": UNITS[wl], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    if wl == "augment":
        boxes, flips = golden_boxes(AUG_B)
        try:
            from oracle import swscale_ref as SW

            per_step = AUG_B                        # one step = the config's whole 64-clip batch
            sws = SW.load()
            if sws is None:
                raise RuntimeError("no libswscale")
            from concurrent.futures import ThreadPoolExecutor

            rng = np.random.default_rng(0)
            frames = [rng.integers(0, 256, (AUG_T, AUG_H, AUG_W, 3), dtype=np.uint8) for _ in range(2)]

            def job(i):
                return SW.scale_clip(sws, frames[i % 2], boxes[i % len(boxes)], bool(flips[i % len(flips)]))

            what = (f"one {per_step}-clip batch per step: crop -> hflip -> sws_scale(SWS_BILINEAR|SWS_ACCURATE_RND) "
                    f"320x568 -> 224^2 per frame (codec.cpp:226-246) via ctypes on {SW.version_tag()}, "
                    f"{cores} clips in flight; no normalise/cast (the reference defers them)")
            ex = ThreadPoolExecutor(cores)
            for w in range(args.warmup):
                list(ex.map(job, range(w * per_step, (w + 1) * per_step)))
            t0 = time.perf_counter()
            for s_ in range(args.steps):
                list(ex.map(job, range(s_ * per_step, (s_ + 1) * per_step)))
            sec = time.perf_counter() - t0
            ex.shutdown()
            v = per_step * args.steps / sec
            kind, dtype = "reference", "u8"
        except RuntimeError:
            from oracle import cpu_baseline as CB
            import torch

            torch.set_num_threads(cores)
            g = torch.Generator().manual_seed(0)
            fr = torch.randint(0, 256, (2, AUG_T, AUG_H, AUG_W, 3), generator=g, dtype=torch.uint8)
            per_step = 2
            for w in range(args.warmup):
                CB.transform_clip_torch(fr[w % 2], boxes[w % len(boxes)], bool(flips[w % len(flips)]))
            t0 = time.perf_counter()
            for s_ in range(args.steps * per_step):
                CB.transform_clip_torch(fr[s_ % 2], boxes[s_ % len(boxes)], bool(flips[s_ % len(flips)]))
            sec = time.perf_counter() - t0
            v = per_step * args.steps / sec
            kind, dtype, what = "port", "f32", f"{per_step} clips per step, torch fp32 restatement"
        return dict(base, value=v, ms_per_step=sec / args.steps * 1e3, dtype=dtype,
                    data="synthetic uint8 clips, reference sampler boxes",
                    cpu_baseline={"value": v, "unit": UNITS[wl], "cores": cores, "kind": kind, "sample": what},
                    e2e={"value": v, "unit": UNITS[wl], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    # training workloads: one real fp32 training step of the restatement per bench step
    from oracle import vit_oracle as VO
    from paper_2309_16669_b200.vit import CONFIG3_VIT_B, CONFIG4_VIT_B_16F, CONFIG5_VIT_L_16F, TextConfig

    if wl == "clip":
        per_step = 2               # the smallest batch with a contrastive term
        st = VO.CpuTrainStep(CONFIG3_VIT_B, per_step, cores, kind="clip", tcfg=TextConfig())
        what = f"{per_step} pairs per step: fp32 CLIP dual-encoder fwd+bwd+AdamW (oracle/vit_oracle.py)"
    else:
        per_step = 1
        cfg = CONFIG5_VIT_L_16F if wl == "train-l14" else CONFIG4_VIT_B_16F
        st = VO.CpuTrainStep(cfg, per_step, cores, kind="finetune", num_classes=3806)
        what = f"{per_step} clip per step: fp32 fine-tune fwd+bwd+AdamW (oracle/vit_oracle.py)"
    for _ in range(args.warmup):
        st.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        st.step()
    sec = time.perf_counter() - t0
    v = per_step * args.steps / sec
    return dict(base, value=v, ms_per_step=sec / args.steps * 1e3, dtype="f32",
                data="synthetic clips, random-init weights",
                cpu_baseline={"value": v, "unit": UNITS[wl], "cores": cores, "kind": "port",
                              "sample": what + f", {cores} threads (the reference has no encoder code; SURVEY 8(c))"},
                e2e={"value": v, "unit": UNITS[wl], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})


def _relaunch(args) -> None:
    """--gpus N > 1 outside a launcher: re-exec under torch.distributed.run with N local ranks."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # communicator lines show the N ranks (on stderr)
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execvpe(sys.executable, cmd, env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="train", choices=list(METRICS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-breakdown", action="store_true", help="skip the per-kernel breakdown pass")
    ap.add_argument("--eager", action="store_true", help="no CUDA-graph replay of the training step")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch(args)

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    rank, world, local = dist_setup(args.gpus)
    if args.workload == "augment":
        line = run_augment(args, rank, world, local)
    elif args.workload == "feed":
        line = run_feed(args, rank, world, local)
    elif args.workload == "clip":
        from paper_2309_16669_b200 import clip_bench

        line = clip_bench.run(args, rank, world, local, ClockSampler, barrier, max_over_ranks, peaks)
    else:
        from paper_2309_16669_b200 import train_bench

        line = train_bench.run(args, rank, world, local, ClockSampler, barrier, max_over_ranks, peaks,
                               large=(args.workload == "train-l14"))
    line["metric"] = METRICS[args.workload]
    line["config"] = workload_config(args.workload, world)     # identical to the reference arm's
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
