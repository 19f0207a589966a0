"""Per-key-tile event timeline of K4 for CTA (0,0,0) on the config-4 shape (AVB_ATTN_FTRACE debug hook).
Needs a build with the hooks compiled in:
  AVB_NVCC_DEFS=-DAVB_ATTN_TRACE_HOOKS python -c "from paper_2309_16669_b200 import build as B; B.build(clean=True)"
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
B, N, H = 64, 1569, 12
tr = torch.zeros(64 * 16, dtype=torch.int64, device="cuda")
os.environ["AVB_ATTN_FTRACE"] = str(tr.data_ptr())
from paper_2309_16669_b200 import ops
D = H * 64
qkv = (torch.randn(B, N, 3 * D, device="cuda") * 0.5).to(torch.bfloat16)
q, k, v = qkv[:, :, :D], qkv[:, :, D:2 * D], qkv[:, :, 2 * D:]
for _ in range(3):
    o, lse = ops.attn_fwd(q, k, v, H)
torch.cuda.synchronize()
t = tr.view(64, 16).cpu()
t0 = int(t[0, 9])
names = {9: "tma", 3: "g0:s_full", 4: "g0:max", 5: "g0:o_full", 6: "g0:p_arr", 7: "g1:s_full", 8: "g1:p_arr",
         0: "m:wait_p0", 1: "m:iss0", 10: "m:wait_p1", 2: "m:iss1"}
for j in [int(x) for x in os.environ.get("TRACE_TILES", "0,1,2,10,11,12,24").split(",")]:
    print(j, "  ".join(f"{names[e]}={int(t[j, e]) - t0}" for e in (9, 3, 4, 5, 6, 7, 8, 0, 1, 10, 2) if int(t[j, e]) != 0))
tops = [int(t[j, 3]) for j in range(25) if int(t[j, 3])]
print("g0 s_full deltas:", [b - a for a, b in zip(tops, tops[1:])])
