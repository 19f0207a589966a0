"""bench.py --workload clip: BASELINE.json configs[2], ViT-B/16 CLIP dual encoder.

Per GPU: 128 clips of 4x224^2 (K1 from decoded uint8 4x320x568 clips, tubelet 1x16x16 -> N=785)
+ 128 captions x 77 tokens (12-layer, width-512 causal text tower), projection 256, one fused
[B, 512] embedding all_gather -> InfoNCE over the global batch (1024 at 8 GPUs) -> local-row
gradients -> bucketed gradient all-reduce overlapped with the backward -> AdamW.  Weak scaling.
"""

from __future__ import annotations

import numpy as np
import torch

from .clip import CLIPModel
from .dp import GradBucketReducer
from .train_bench import golden_boxes

PAIRS_PER_GPU = 128
SRC_T, SRC_H, SRC_W = 4, 320, 568


def run(args, rank, world, local, ClockSampler, barrier, max_over_ranks, peaks):
    from . import transform as TR

    dev = torch.device("cuda", torch.cuda.current_device())
    model = CLIPModel(device=dev, seed=0)
    vc, tcfg = model.vcfg, model.tcfg
    B = PAIRS_PER_GPU
    boxes, flips = golden_boxes(B, offset=rank * B)
    g = torch.Generator(device=dev).manual_seed(4321 + rank)
    frames = torch.randint(0, 256, (B, SRC_T, SRC_H, SRC_W, 3), generator=g, dtype=torch.uint8, device=dev)
    tokens = torch.randint(0, tcfg.vocab, (B, tcfg.context), generator=g, device=dev, dtype=torch.int32)
    eot_pos = np.random.default_rng(rank).integers(5, tcfg.context, B)       # caption lengths (host-side data)
    eot = torch.from_numpy((np.arange(B) * tcfg.context + eot_pos).astype(np.int32)).to(dev)
    boxes_d = torch.from_numpy(boxes).to(dev)
    flips_d = torch.from_numpy(flips).to(dev)
    patches = torch.empty((B * vc.patches, vc.patch_dim), dtype=torch.bfloat16, device=dev)
    loss = torch.zeros(1, device=dev)
    store = model.store
    reducer = GradBucketReducer(store.grad, {gname: store.group_slice(gname) for gname in store.groups})

    def k1():
        TR.transform(frames, boxes_d, flips_d, (vc.height, vc.width), out=patches, layout="tubelet", crops_host=boxes,
                     tubelet=(vc.cube_t, vc.cube_h, vc.cube_w), validate=False)

    def model_step():
        store.grad.zero_()
        loss.zero_()
        model.forward_backward(patches, tokens, eot, loss, on_layer_done=reducer.on_layer_done)
        reducer.finish()
        model.optimizer_step(grad_scale=1.0 / world)

    def eager_step():
        k1()
        model_step()

    # breakdown pass first (eager, CUDA events around every launch), then the graph takes its own pool
    from .train_bench import instrumented_pass

    for _ in range(args.warmup):
        eager_step()
    nb = 0 if args.no_breakdown else 2
    fam, lps = instrumented_pass(eager_step, nb)

    # single process: both towers' step replays from one captured CUDA graph (as the train workload)
    graphed = None
    if world == 1 and not args.eager:
        from .vit import CapturedStep

        k1()
        graphed = CapturedStep(model_step, warmup=args.warmup)

    def step():
        if graphed is None:
            eager_step()
        else:
            k1()
            graphed()

    for _ in range(args.warmup):
        step()
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

    host = torch.empty((B, SRC_T, SRC_H, SRC_W, 3), dtype=torch.uint8, pin_memory=True)
    host.copy_(frames.cpu())
    tok_h = tokens.cpu().pin_memory()
    loss_h = torch.empty(1, dtype=torch.float32, pin_memory=True)

    def e2e_step():
        frames.copy_(host, non_blocking=True)
        tokens.copy_(tok_h, non_blocking=True)
        step()
        loss_h.copy_(loss, non_blocking=True)

    for _ in range(2):
        e2e_step()
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    flops = B * world * 3.0 * (vc.forward_flops_per_clip() + 2.0 * tcfg.context * tcfg.dim * tcfg.dim * 12 *
                                tcfg.depth + 4.0 * tcfg.context ** 2 * tcfg.dim * tcfg.depth)
    pk, src = peaks()
    # the dominant kernel of the breakdown pass: its achieved rate = the roofline
    roof = None
    if fam:
        N, Hh = vc.tokens, vc.heads
        att_f = 4.0 * B * Hh * N * N * 64
        cands = {}
        for k, v in fam.items():
            if k.startswith("gemm:"):
                dims = k.split(":")[1].split("/")[0].split("x")
                cands[k] = (v["total_ms"] / nb, 2.0 * int(dims[0]) * int(dims[1]) * int(dims[2]) / (v["avg_ms"] / 1e3))
        # video-tower attention launches: the fwd/bwd families mix video (N=785) and text (L=77) layers,
        # the video ones dominate (12 x 785^2 vs 12 x 77^2 per clip)
        if "attn_bwd" in fam:
            cands["attn_bwd"] = (fam["attn_bwd"]["total_ms"] / nb,
                                 2 * att_f * vc.depth / (fam["attn_bwd"]["total_ms"] / nb / 1e3))
        if "attn_fwd" in fam:
            cands["attn_fwd"] = (fam["attn_fwd"]["total_ms"] / nb,
                                 att_f * vc.depth / (fam["attn_fwd"]["total_ms"] / nb / 1e3))
        dom = max(cands, key=lambda k: cands[k][0])
        ach = cands[dom][1] / 1e12
        roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": pk["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": ach / pk["bf16_tflops_sustained"], "traffic": None,
                "share_of_step": cands[dom][0] / ms,
                "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside a long step)"}
    line = {
        "metric": "train pairs/sec ViT-B/16 CLIP dual encoder 4x224^2, InfoNCE over the global batch",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic uint8 4x320x568 clips + random 77-token captions; random-init weights",
        "config": {"workload": "configs[2] ViT-B/16 CLIP dual encoder 4x224^2 (N=785) + 12L/512 text, proj 256",
                   "pairs_per_gpu": B, "global_batch": B * world, "parallelism": f"dp{world}"},
        "model_tflops": flops / (ms / 1e3) / 1e12 / world,
        "execution": ("K1 launch + both towers' step replayed from one captured CUDA graph" if graphed is not None
                      else "eager launches"),
        "e2e": {"value": B * world / (e2e_ms / 1e3), "unit": "pairs/s",
                "h2d_bytes_per_step": int(host.numel() + tok_h.numel() * 4), "d2h_bytes_per_step": 4},
        "clocks": clocks, "loss": float(loss_h.item()),
        "roofline": roof,
        "kernels": {k: v for k, v in fam.items() if ":" not in k},
        "gpu_launches": (lps * args.steps) if lps else None,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import os

        from oracle import vit_oracle as VO

        cores = os.cpu_count() or 1
        st = VO.CpuTrainStep(vc, 2, cores, kind="clip", tcfg=tcfg)
        st.step()
        import time

        t0 = time.perf_counter()
        st.step()
        sec = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": 2.0 / sec, "unit": "pairs/s", "cores": cores, "kind": "port",
                                "sample": "2 pairs, one fp32 CLIP dual-encoder fwd+bwd+AdamW step of the torch "
                                          "restatement (oracle/vit_oracle.py), all host threads"}
    return line
