"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic.

* GradBucketReducer: per-layer slices all-reduced asynchronously in backward order equal the
  plain sum; untouched slices stay local.
* gather_embeddings + the CLIP gradient rule: every rank evaluates
  the loss on the gathered global batch but back-propagates only its own rows; scaling the
  local encoder gradients by world and MEAN-reducing reproduces the single-process gradient,
  and the replicated logit-scale gradient survives the mean unchanged.  The loss math is the
  oracle's (oracle/vit_oracle.clip_loss); the fused GPU kernel's local-row gradients are
  checked against the same oracle in tests/test_infonce_gpu.py.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reducer_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_16669_b200.dp import GradBucketReducer
        flat = torch.arange(20, dtype=torch.float32) * (rank + 1)
        slices = {"head": (15, 20), "blk1": (8, 15), "blk0": (2, 8), "embed": (0, 2)}
        red = GradBucketReducer(flat, slices)
        for name in ["head", "blk1", "blk0"]:          # 'embed' deliberately not reduced
            red.on_layer_done(name)
        done = red.finish()
        q.put((rank, flat.tolist(), done))
    finally:
        dist.destroy_process_group()


def _clip_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import vit_oracle as VO
        from paper_2309_16669_b200 import dp
        g = torch.Generator().manual_seed(0)
        B, E = 3, 8
        W = torch.randn(E, 5, generator=g)                  # shared "encoder" weight
        xs = torch.randn(world * B, 5, generator=g)         # all clips; rank takes its rows
        ys = torch.randn(world * B, 5, generator=g)
        scale = torch.tensor(1 / 0.07)
        Wl = W.clone().requires_grad_(True)
        sl = scale.clone().requires_grad_(True)
        v_loc = xs[rank * B:(rank + 1) * B] @ Wl.t()
        t_loc = ys[rank * B:(rank + 1) * B] @ Wl.t()
        v_all, t_all = dp.gather_embeddings(v_loc.detach(), t_loc.detach())
        r0, n = dp.local_rows(B)
        # keep only the local rows attached to the graph
        v_cat = torch.cat([v_all[:r0], v_loc, v_all[r0 + n:]])
        t_cat = torch.cat([t_all[:r0], t_loc, t_all[r0 + n:]])
        loss = VO.clip_loss(v_cat, t_cat, sl)
        loss.backward()
        gW = Wl.grad * dp.local_grad_scale()
        dist.all_reduce(gW)
        gW /= world
        gs = sl.grad.clone()
        dist.all_reduce(gs)
        gs /= world
        q.put((rank, gW, gs, loss.item()))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_bucket_reducer_gloo():
    res = _run(_reducer_worker)
    base = torch.arange(20, dtype=torch.float32)
    for rank, flat, done in res:
        flat = torch.tensor(flat)
        assert done == ["head", "blk1", "blk0"]
        assert torch.allclose(flat[2:], base[2:] * 3)          # (1 + 2) summed over ranks
        assert torch.allclose(flat[:2], base[:2] * (rank + 1))  # not reduced


def test_clip_dp_gradient_rule_gloo():
    from oracle import vit_oracle as VO
    res = _run(_clip_worker)
    # single-process reference over the same global batch
    g = torch.Generator().manual_seed(0)
    W = torch.randn(8, 5, generator=g)
    xs = torch.randn(6, 5, generator=g)
    ys = torch.randn(6, 5, generator=g)
    Wr = W.clone().requires_grad_(True)
    sr = torch.tensor(1 / 0.07, requires_grad=True)
    loss = VO.clip_loss(xs @ Wr.t(), ys @ Wr.t(), sr)
    loss.backward()
    for rank, gW, gs, l in res:
        assert abs(l - loss.item()) < 1e-5
        assert torch.allclose(gW, Wr.grad, atol=1e-5, rtol=1e-4)
        assert torch.allclose(gs, sr.grad, atol=1e-6)


# ----------------------------------------------------------------------------- the real DP step (GPU)
def _ft_worker(rank, world, port, q):
    """One rank of the data-parallel fine-tune step: its half of the clips, gradients all-reduced
    per layer through GradBucketReducer while the backward runs (gloo carries CUDA tensors, so two
    ranks can share the one GPU of the test box; the bench uses NCCL)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_16669_b200.dp import GradBucketReducer
        cfg, C, B, patches, labels = _ft_inputs()
        from paper_2309_16669_b200.vit import FineTuneModel
        model = FineTuneModel(cfg, num_classes=C, seed=1)
        s = model.store
        red = GradBucketReducer(s.grad, {g: s.group_slice(g) for g in s.groups})
        half = B // world
        Np = cfg.patches
        loss = torch.zeros(1, device="cuda")
        model.zero_grad()
        model.forward_backward(patches[rank * half * Np:(rank + 1) * half * Np].contiguous(),
                               labels[rank * half:(rank + 1) * half].contiguous(), half, loss,
                               loss_scale=1.0 / B, on_layer_done=red.on_layer_done)
        done = red.finish()
        torch.cuda.synchronize()
        q.put((rank, s.grad.cpu(), done))
    finally:
        dist.destroy_process_group()


def _ft_inputs():
    from paper_2309_16669_b200.vit import VitConfig
    cfg = VitConfig(frames=4, height=64, width=64, cube_t=2, depth=2, dim=128, heads=2)
    C, B = 10, 4
    g = torch.Generator(device="cuda").manual_seed(7)
    patches = torch.randn(B * cfg.patches, cfg.patch_dim, generator=g, device="cuda").to(torch.bfloat16)
    labels = torch.randint(0, C, (B,), generator=g, device="cuda", dtype=torch.int32)
    return cfg, C, B, patches, labels


@pytest.mark.gpu
def test_dp_finetune_step_equals_single_rank_2x_batch():
    from paper_2309_16669_b200.vit import FineTuneModel
    res = _run(_ft_worker)
    cfg, C, B, patches, labels = _ft_inputs()
    model = FineTuneModel(cfg, num_classes=C, seed=1)
    loss = torch.zeros(1, device="cuda")
    model.zero_grad()
    model.forward_backward(patches, labels, B, loss, loss_scale=1.0 / B)
    ref = model.store.grad.cpu()
    st = model.store
    for rank, grad, done in res:
        assert "head" in done and "enc.embed" in done and len(done) == cfg.depth + 2
        # same kernels on half the clips each + the sum over ranks == one rank on all clips
        per = {}
        for name in st.groups:
            a, b = st.group_slice(name)
            per[name] = ((grad[a:b] - ref[a:b]).norm() / ref[a:b].norm().clamp_min(1e-30)).item()
        tot = ((grad - ref).norm() / ref.norm()).item()
        if os.environ.get("AVB_TEST_VERBOSE"):
            print("dp rel", rank, f"{tot:.3e}", {k: f"{v:.1e}" for k, v in per.items()})
        assert tot < 1e-3, (rank, per)


def test_bench_self_launch_command(monkeypatch):
    """`bench.py --gpus N` outside a launcher re-executes itself under torch.distributed.run."""
    import sys
    import bench
    seen = {}
    monkeypatch.setattr(bench.os, "execvpe", lambda f, cmd, env: seen.update(cmd=cmd, env=env))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5"])

    class A:
        gpus = 4
    bench._relaunch(A())
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "5"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
