"""K1 alone at config 2 (64 clips 16x320x568 -> bf16 16x224^2, reference-sampler boxes): ms and GB/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2309_16669_b200 import transform as TR

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
g = np.asarray(json.load(open(os.path.join(ROOT, "tests", "golden", "rrc_golden.json")))["config2_568x320"], np.int32)
B = 64
boxes, flips = np.ascontiguousarray(g[:B, :4]), np.ascontiguousarray(g[:B, 4].astype(np.uint8))
fr = torch.randint(0, 256, (B, 16, 320, 568, 3), dtype=torch.uint8, device="cuda")
bd, fd = torch.from_numpy(boxes).cuda(), torch.from_numpy(flips).cuda()
res = {}
for layout, shape in (("cthw", (B, 3, 16, 224, 224)), ("tubelet", (B * 8 * 14 * 14, 1536))):
    out = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    kw = dict(layout=layout, crops_host=boxes, tubelet=(2, 16, 16), validate=False)
    for _ in range(3):
        TR.transform(fr, bd, fd, out=out, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        TR.transform(fr, bd, fd, out=out, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    algo = TR.algorithmic_bytes(boxes, 16, (224, 224), 2)
    res[layout] = {"ms": ms, "GBs": algo / ms / 1e6}
# the reference loader's planar layout [B,T,3,H,W] with crops (v4 with one bulk copy per channel plane)
planar = fr.permute(0, 1, 4, 2, 3).contiguous()
out = torch.empty((B, 3, 16, 224, 224), dtype=torch.bfloat16, device="cuda")
kw = dict(layout="cthw", crops_host=boxes, validate=False, channels_last=False)
for _ in range(2):
    TR.transform(planar, bd, fd, out=out, **kw)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    TR.transform(planar, bd, fd, out=out, **kw)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
res["planar"] = {"ms": ms, "GBs": TR.algorithmic_bytes(boxes, 16, (224, 224), 2) / ms / 1e6}
print(json.dumps(res))
