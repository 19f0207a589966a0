"""bench.py --workload train: BASELINE.json configs[3], ViT-B/16 fine-tune 16x224^2 (N=1569).

One step per GPU = K1 (decoded uint8 clips -> tubelet patch rows, bf16) + encoder forward
+ cls head CE + full backward + (N>1: bucketed NCCL all-reduce of gradients, overlapped
with the backward as each layer's slice becomes final) + fused AdamW.  64 clips per GPU
(PAPER.md:1207), weak scaling.
"""

from __future__ import annotations

import json
import os

import numpy as np
import torch

from . import ops
from .vit import CONFIG4_VIT_B_16F, CONFIG5_VIT_L_16F, FineTuneModel

CLIPS_PER_GPU = 64
ATTN_BWD_LAUNCHES = 2    # avb_attn_bwd = delta/lse prologue (+ dQ zeroing) + K5
NUM_CLASSES = 3806
SRC_T, SRC_H, SRC_W = 16, 320, 568


class LaunchTimer:
    """CUDA-event brackets around selected kernel families inside the timed region."""

    def __init__(self):
        self.ev = {}
        self.active = False

    def wrap(self, name, fn, keyfn=None):
        def inner(*a, **k):
            if not self.active:
                return fn(*a, **k)
            s = torch.cuda.current_stream()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            r = fn(*a, **k)
            e1.record(s)
            self.ev.setdefault(name, []).append((e0, e1))
            if keyfn is not None:
                self.ev.setdefault(name + ":" + keyfn(*a, **k), []).append((e0, e1))
            return r
        return inner

    def summary(self):
        out = {}
        for k, lst in self.ev.items():
            ms = [a.elapsed_time(b) for a, b in lst]
            out[k] = {"launches": len(ms), "total_ms": float(np.sum(ms)), "avg_ms": float(np.mean(ms))}
        return out


def golden_boxes(n: int, offset: int = 0):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "tests", "golden", "rrc_golden.json")) as fh:
        g = np.asarray(json.load(fh)["config2_568x320"], dtype=np.int32)
    idx = (np.arange(n) + offset) % len(g)
    return np.ascontiguousarray(g[idx, :4]), np.ascontiguousarray(g[idx, 4].astype(np.uint8))


INSTRUMENTED = ("attn_fwd", "attn_bwd", "gemm", "layernorm_fwd", "layernorm_bwd", "colsum_accum", "tokens_fwd",
                "tokens_bwd", "xent", "adamw", "infonce_fwd", "infonce_bwd", "embed_fwd", "embed_bwd", "rows_copy",
                "cast_bf16", "patchify")


def gemm_key(a, b, a_mn=False, b_mn=False, epilogue=0, split_k=1, **k):
    M, K = (a.shape[1], a.shape[0]) if a_mn else (a.shape[0], a.shape[1])
    N = b.shape[1] if b_mn else b.shape[0]
    return f"{M}x{N}x{K}/{'T' if a_mn else 'N'}{'T' if b_mn else 'N'}/epi{epilogue}/s{split_k}"


def instrumented_pass(step, nb: int):
    """Run `step` nb more times with CUDA events around every ops.* launch and K1 (`transform`):
    returns (per-family timing summary, kernel launches per step, the grad memset included).
    Used AFTER the timed region, never inside it."""
    from . import transform as TR

    if nb <= 0:
        return {}, None
    timer = LaunchTimer()
    counts = {"n": 0}
    orig = {n: getattr(ops, n) for n in INSTRUMENTED}
    orig_tr = TR.transform
    per_launch = {"attn_bwd": ATTN_BWD_LAUNCHES, "infonce_fwd": 3}

    def counted(name, fn):
        def inner(*a, **k):
            counts["n"] += per_launch.get(name, 1)
            return fn(*a, **k)
        return inner

    try:
        for n, fn in orig.items():
            setattr(ops, n, timer.wrap(n, counted(n, fn), keyfn=gemm_key if n == "gemm" else None))
        TR.transform = timer.wrap("k1_transform", counted("k1_transform", orig_tr))
        timer.active = True
        for _ in range(nb):
            counts["n"] += 1      # the gradient memset
            step()
        torch.cuda.synchronize()
    finally:
        timer.active = False
        for n, fn in orig.items():
            setattr(ops, n, fn)
        TR.transform = orig_tr
    return timer.summary(), counts["n"] // nb


def traffic(kernel: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture (or None)."""
    import bench  # noqa: the driver script's helper (profiles/r01/traffic.json)

    return bench.ncu_traffic(kernel)


def run(args, rank, world, local, ClockSampler, barrier, max_over_ranks, peaks, large: bool = False):
    """large=False: configs[3] ViT-B/16 (64 clips/GPU); large=True: configs[4] ViT-L/14 (24 clips/GPU)."""
    cfg = CONFIG5_VIT_L_16F if large else CONFIG4_VIT_B_16F
    B = 24 if large else CLIPS_PER_GPU
    dev = torch.device("cuda", torch.cuda.current_device())
    model = FineTuneModel(cfg, NUM_CLASSES, device=dev, seed=0)   # identical init on every rank
    boxes, flips = golden_boxes(B, offset=rank * B)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    frames = torch.randint(0, 256, (B, SRC_T, SRC_H, SRC_W, 3), generator=g, dtype=torch.uint8, device=dev)
    labels = torch.randint(0, NUM_CLASSES, (B,), generator=g, device=dev, dtype=torch.int32)
    boxes_d = torch.from_numpy(boxes).to(dev)
    flips_d = torch.from_numpy(flips).to(dev)
    patches = torch.empty((B * cfg.patches, cfg.patch_dim), dtype=torch.bfloat16, device=dev)
    loss = torch.zeros(1, dtype=torch.float32, device=dev)

    from .dp import GradBucketReducer

    store = model.store
    reducer = GradBucketReducer(store.grad, {g: store.group_slice(g) for g in store.groups})
    on_layer_done = reducer.on_layer_done

    from . import transform as TR

    def k1(*a, **k):
        return TR.transform(*a, **k)

    def zero():
        store.grad.zero_()

    def eager_step():
        zero()
        loss.zero_()
        k1(frames, boxes_d, flips_d, (cfg.height, cfg.width), out=patches, layout="tubelet", crops_host=boxes,
           tubelet=(cfg.cube_t, cfg.cube_h, cfg.cube_w), validate=False)
        model.forward_backward(patches, labels, B, loss, on_layer_done=on_layer_done)
        reducer.finish()
        model.optimizer_step(grad_scale=1.0 / world)

    # ---- breakdown pass (separate from the timed region, run first so its eager allocations are all
    # cached before the graph below takes its own pool): CUDA events around every kernel family and a
    # launch counter; its shares explain `value`, they are not part of it
    for _ in range(args.warmup):
        eager_step()
    nb = 0 if args.no_breakdown else max(2, min(args.steps, 4))
    fam, launches_per_step = instrumented_pass(eager_step, nb)

    # single process: the model part of the step (everything after K1) replays from one captured CUDA
    # graph; with N ranks the step stays eager (the DP all-reduce overlaps the backward on NCCL's stream)
    graphed = None
    if world == 1 and not args.eager:
        k1(frames, boxes_d, flips_d, (cfg.height, cfg.width), out=patches, layout="tubelet", crops_host=boxes,
           tubelet=(cfg.cube_t, cfg.cube_h, cfg.cube_w), validate=False)
        graphed = model.capture_train_step(patches, labels, B, loss, warmup=args.warmup)

    def step():
        if graphed is None:
            eager_step()
            return
        k1(frames, boxes_d, flips_d, (cfg.height, cfg.width), out=patches, layout="tubelet", crops_host=boxes,
           tubelet=(cfg.cube_t, cfg.cube_h, cfg.cube_w), validate=False)
        graphed()

    for _ in range(args.warmup):
        step()
    # ---- the timed region: K plain steps, no per-launch instrumentation of any kind
    barrier(world)
    clk = ClockSampler(local)
    clk.start()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = clk.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    value = B * world / (ms / 1e3)


    N, H = cfg.tokens, cfg.heads
    att_f = 4.0 * B * H * N * N * 64                    # per launch (one layer)
    att_b = 2.0 * att_f                                 # algorithmic (3x fwd convention, no recompute)
    pk, src = peaks()
    gemm_flops_step = B * (cfg.forward_flops_per_clip() - cfg.attention_forward_flops_per_clip()) * 3.0
    kern = {}
    if "attn_fwd" in fam:
        kern["attn_fwd"] = dict(fam["attn_fwd"], tflops=att_f / (fam["attn_fwd"]["avg_ms"] / 1e3) / 1e12)
    if "attn_bwd" in fam:
        kern["attn_bwd"] = dict(fam["attn_bwd"], tflops=att_b / (fam["attn_bwd"]["avg_ms"] / 1e3) / 1e12)
    if "gemm" in fam:
        gms = fam["gemm"]["total_ms"] / nb
        kern["gemm_all"] = dict(fam["gemm"], tflops=gemm_flops_step / (gms / 1e3) / 1e12)
    for k, v in fam.items():
        if ":" not in k and k not in ("attn_fwd", "attn_bwd", "gemm"):
            kern[k] = dict(v)
    for k in kern:
        kern[k]["share_of_step"] = kern[k]["total_ms"] / nb / ms
    shapes = {}
    for k, v in fam.items():
        if k.startswith("gemm:"):
            dims = k.split(":")[1].split("/")[0].split("x")
            fl = 2.0 * int(dims[0]) * int(dims[1]) * int(dims[2])
            shapes[k[5:]] = {"ms_per_step": v["total_ms"] / nb, "launches_per_step": v["launches"] / nb,
                             "tflops": fl / (v["avg_ms"] / 1e3) / 1e12}
    shapes = dict(sorted(shapes.items(), key=lambda kv: -kv[1]["ms_per_step"])[:16])
    roof = None
    if kern:
        # dominant single kernel: attention fwd/bwd are one kernel each; GEMM instantiations split per shape
        cands = {k: kern[k]["total_ms"] / nb for k in ("attn_fwd", "attn_bwd") if k in kern}
        for k, v in shapes.items():
            cands["gemm:" + k] = v["ms_per_step"]
        dom = max(cands, key=cands.get)
        ach = shapes[dom[5:]]["tflops"] if dom.startswith("gemm:") else kern[dom]["tflops"]
        roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": pk["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": ach / pk["bf16_tflops_sustained"],
                "traffic": None if large else traffic(dom),   # the committed capture is of the config-4 shape
                "share_of_step": cands[dom] / ms,
                "algorithmic_flops_per_launch": (att_b if dom == "attn_bwd" else att_f if dom == "attn_fwd" else None),
                "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside a long step)"}
    attn_total_ms = sum(kern[k]["total_ms"] for k in ("attn_fwd", "attn_bwd") if k in kern) / max(nb, 1)
    attn_tflops = (att_f + att_b) * cfg.depth / (attn_total_ms / 1e3) / 1e12 if attn_total_ms else None
    k1_roof = None
    if "k1_transform" in fam:
        algo = TR.algorithmic_bytes(boxes, SRC_T, (cfg.height, cfg.width), 2)
        gbs = algo / (fam["k1_transform"]["avg_ms"] / 1e3) / 1e9
        k1_roof = {"bound": "hbm", "kernel": "k1v4_kernel (tubelet layout)", "achieved": gbs, "peak": pk["hbm_gbs"],
                   "unit": "GB/s", "frac": gbs / pk["hbm_gbs"], "algorithmic_bytes_per_launch": algo,
                   "ms_per_launch": fam["k1_transform"]["avg_ms"], "peak_source": f"{src} hbm_gbs (in-step)"}

    # ---- e2e: public API from pinned host clips; every step's clips cross H2D inside the timed region.
    # Loader -> device hand-off: the next step's clips are copied on a side
    # stream into the other half of a double buffer while the current step computes.
    host = torch.empty((B, SRC_T, SRC_H, SRC_W, 3), dtype=torch.uint8, pin_memory=True)
    host.copy_(frames.cpu())
    loss_h = torch.empty(1, dtype=torch.float32, pin_memory=True)
    from .feeder import DeviceFeeder

    feeder = DeviceFeeder(B, SRC_T, SRC_H, SRC_W, (cfg.height, cfg.width), layout="tubelet",
                          tubelet=(cfg.cube_t, cfg.cube_h, cfg.cube_w), channels_last=True, depth=2)

    def e2e_run(nsteps):
        # public API: the feeder H2D-copies step i+1's pinned clips on its copy stream while step i computes
        feeder.submit(host, boxes, flips)
        for i in range(nsteps):
            if i + 1 < nsteps:
                feeder.submit(host, boxes, flips)
            feeder.next(out=patches)
            if graphed is not None:
                graphed()
            else:
                zero()
                loss.zero_()
                model.forward_backward(patches, labels, B, loss, on_layer_done=on_layer_done)
                reducer.finish()
                model.optimizer_step(grad_scale=1.0 / world)
            loss_h.copy_(loss, non_blocking=True)

    e2e_run(2)
    torch.cuda.synchronize()
    barrier(world)
    e0.record(stream)
    e2e_run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)

    line = {
        "metric": None,   # bench.py sets the workload's shared metric string and config
        "value": value, "unit": "clips/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic uint8 16x320x568 clips (device randint) -> K1 RRC boxes from the reference sampler; "
                "random-init weights; random labels over 3806 classes",
        "attn_tflops": attn_tflops,
        "kernels": kern,
        "gemm_shapes": shapes,
        "roofline": roof,
        "k1_roofline": k1_roof,
        "breakdown": f"{nb} extra eager steps before the timed region with CUDA events around every launch",
        "execution": ("K1 launch + the model step replayed from one captured CUDA graph" if graphed is not None
                      else "eager launches"),
        "e2e": {"value": B * world / (e2e_ms / 1e3), "unit": "clips/s", "h2d_bytes_per_step": int(host.numel()),
                "d2h_bytes_per_step": 4},
        "gpu_launches": (launches_per_step * args.steps) if launches_per_step else None,
        "clocks": clocks,
        "loss": float(loss_h.item()),
        "memory": {"peak_bytes": int(torch.cuda.max_memory_allocated()), "clips_per_gpu": B},
    }
    try:  # the reference planners fed with this measurement
        from .perf_models import b200_report

        line["pipeline_model"] = b200_report({"value": line["value"], "n_gpus": world, "memory": line["memory"]}, cfg)
    except Exception as e:  # noqa: BLE001 -- a planner failure must not void the measurement
        line["pipeline_model"] = f"unavailable: {e}"
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import vit_oracle as VO

        cores = os.cpu_count() or 1
        sec = VO.cpu_train_step_time(cfg, NUM_CLASSES, 1, cores, steps=1)
        line["cpu_baseline"] = {"value": 1.0 / sec, "unit": "clips/s", "cores": cores, "kind": "port",
                                "sample": "1 clip, one fp32 fwd+bwd+AdamW step of the torch restatement "
                                          "(oracle/vit_oracle.py), all host threads"}
    return line
