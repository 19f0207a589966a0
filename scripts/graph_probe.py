"""Probe: the config-4 training step eager vs replayed from one captured CUDA graph (timing only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2309_16669_b200 import transform as TR
from paper_2309_16669_b200.train_bench import CLIPS_PER_GPU, NUM_CLASSES, SRC_H, SRC_T, SRC_W, golden_boxes
from paper_2309_16669_b200.vit import CONFIG4_VIT_B_16F as cfg
from paper_2309_16669_b200.vit import FineTuneModel

B = CLIPS_PER_GPU
model = FineTuneModel(cfg, NUM_CLASSES, seed=0)
boxes, flips = golden_boxes(B)
frames = torch.randint(0, 256, (B, SRC_T, SRC_H, SRC_W, 3), dtype=torch.uint8, device="cuda")
labels = torch.randint(0, NUM_CLASSES, (B,), device="cuda", dtype=torch.int32)
bd, fd = torch.from_numpy(boxes).cuda(), torch.from_numpy(flips).cuda()
patches = torch.empty((B * cfg.patches, cfg.patch_dim), dtype=torch.bfloat16, device="cuda")
loss = torch.zeros(1, device="cuda")


def step():
    model.store.grad.zero_()
    loss.zero_()
    TR.transform(frames, bd, fd, (224, 224), out=patches, layout="tubelet", crops_host=boxes, tubelet=(2, 16, 16),
                 validate=False)
    model.forward_backward(patches, labels, B, loss)
    model.optimizer_step()


def timeit(fn, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
print("eager ms", timeit(step))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
print("graph ms", timeit(g.replay))
print("eager ms", timeit(step))
print("graph ms", timeit(g.replay))
