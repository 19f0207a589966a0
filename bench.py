#!/usr/bin/env python
"""Benchmark driver (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload train|augment|clip]

Workloads
  train    (default) BASELINE.json configs[3]: ViT-B/16 fine-tune, 16x224^2 clips,
           tubelet 2x16x16 (N=1569), 64 clips per GPU; one step = K1 augmentation of
           the decoded uint8 clips + encoder fwd/bwd (tcgen05 GEMMs, blockwise
           attention) + CE loss + AdamW; data-parallel over N GPUs (NCCL all-reduce).
  augment  BASELINE.json configs[1]: K1 on 64 synthetic uint8 16x320x568 clips ->
           bf16 16x224^2 with the reference sampler's boxes.
  clip     BASELINE.json configs[2]: ViT-B/16 CLIP dual encoder, 4x224^2 clips + 77-token
           captions, 128 pairs per GPU, embedding all_gather + fused InfoNCE.
  train-l14 BASELINE.json configs[4]: ViT-L/14 16x224^2 (N=2049, D=1024, 24 layers), 24 clips/GPU.

`--impl reference` times the CPU restatement (oracle/, the reference has no GPU
path) on this host's cores, rank 0 only.
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
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


TRAFFIC_PATH = os.path.join(ROOT, "profiles", "r01", "traffic.json")


def ncu_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed `ncu --set full` capture
    (profiles/r01/traffic.json, written by scripts/traffic_from_ncu.py), or None."""
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
    if world > 1:
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
    import torch

    from oracle import cpu_baseline as CB

    cores = os.cpu_count() or 1
    v, n = CB.time_augment(boxes, flips, AUG_T, (AUG_H, AUG_W), budget_s, cores)
    return {"value": v, "unit": "clips/s", "cores": cores, "kind": "port",
            "sample": f"{n} clips x {AUG_T} frames 320x568 -> 224^2, torch fp32 antialiased bilinear "
                      f"restatement + normalize + bf16 cast, torch.set_num_threads({cores})"}


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
        "metric": "augment clips/sec (fused RRC+flip+normalize+bf16, 16x320x568 -> 16x224^2)",
        "value": value, "unit": "clips/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8->bf16",
        "data": "synthetic uint8 clips generated on device (torch.randint, seed=rank); boxes/flips from the "
                "reference sampler (tests/golden/rrc_golden.json)",
        "config": {"workload": "configs[1] fused GPU augmentation", "clips_per_gpu": B, "frames": AUG_T,
                   "src_hw": [AUG_H, AUG_W], "target_hw": [224, 224], "l2": "input 558 MB > 126 MB L2 (no flush)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": ncu_traffic("k1_rrc_normalize"), "peak_source": src,
                     "algorithmic_bytes_per_launch": algo},
        "e2e": {"value": B * world / (e2e_ms / 1e3), "unit": "clips/s",
                "h2d_bytes_per_step": int(host.numel()), "d2h_bytes_per_step": int(res.numel() * 4)},
        "gpu_launches": args.steps,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_augment(boxes, flips)
    return line


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return None
    from oracle import cpu_baseline as CB

    cores = os.cpu_count() or 1
    if args.workload == "augment":
        boxes, flips = golden_boxes(AUG_B)
        vals = []
        for _ in range(args.warmup):
            CB.time_augment(boxes, flips, AUG_T, (AUG_H, AUG_W), 2.0, cores)
        for _ in range(args.steps):
            v, n = CB.time_augment(boxes, flips, AUG_T, (AUG_H, AUG_W), 6.0, cores)
            vals.append(v)
        v = float(np.median(vals))
        return {"impl": "reference", "metric": "augment clips/sec (fused RRC+flip+normalize+bf16, 16x320x568 -> "
                                               "16x224^2)", "value": v, "unit": "clips/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u8->f32->bf16", "data": "synthetic uint8 clips",
                "config": {"workload": "configs[1] fused GPU augmentation", "clips_per_gpu": AUG_B},
                "cpu_baseline": {"value": v, "unit": "clips/s", "cores": cores, "kind": "port",
                                 "sample": "bounded sample of the config-2 batch per step (torch fp32 restatement)"},
                "e2e": {"value": v, "unit": "clips/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return CB.reference_train_line(args, world, cores)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="train", choices=["train", "augment", "clip", "train-l14"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

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
    elif args.workload == "clip":
        from paper_2309_16669_b200 import clip_bench

        line = clip_bench.run(args, rank, world, local, ClockSampler, barrier, max_over_ranks, peaks)
    else:
        from paper_2309_16669_b200 import train_bench

        line = train_bench.run(args, rank, world, local, ClockSampler, barrier, max_over_ranks, peaks,
                               large=(args.workload == "train-l14"))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
