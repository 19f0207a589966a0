"""Per-step event timeline of K5 for CTA (0,0,0) on the config-4 shape (AVB_ATTN_TRACE debug hook).
Needs a build with the hooks compiled in:
  AVB_NVCC_DEFS=-DAVB_ATTN_TRACE_HOOKS python -c "from paper_2309_16669_b200 import build as B; B.build(clean=True)"
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
B, N, H = 64, 1569, 12
tr = torch.zeros(1024 * 32, dtype=torch.int64, device="cuda")
os.environ["AVB_ATTN_TRACE"] = str(tr.data_ptr())
from paper_2309_16669_b200 import ops
D = H * 64
qkv = (torch.randn(B, N, 3 * D, device="cuda") * 0.5).to(torch.bfloat16)
q, k, v = qkv[:, :, :D], qkv[:, :, D:2 * D], qkv[:, :, 2 * D:]
o, lse = ops.attn_fwd(q, k, v, H)
do = torch.randn_like(o)
for _ in range(3):
    ops.attn_bwd(q, k, v, o, do, lse, H)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    ops.attn_bwd(q, k, v, o, do, lse, H)
e1.record(); torch.cuda.synchronize()
print("bwd ms", e0.elapsed_time(e1) / 3)
t = tr.view(1024, 32).cpu()
split = False
t0 = int(t[0, 9 if split else 13])
names = ({0: "m:p_rdy", 1: "m:dV_iss", 2: "m:ds_rdy", 3: "m:dK_iss", 4: "m:dPS_iss", 9: "c:top", 5: "c:s_full",
          6: "c:p_arr", 7: "c:dp_full", 8: "c:ds_arr"} if split else
         {8: "m:wait_p", 0: "m:p_rdy", 9: "m:dV_iss", 10: "m:pt_rd", 11: "m:S_iss", 1: "m:ds_rdy",
          2: "m:dK,dP_iss", 12: "m:dQ_iss", 4: "e:top", 5: "e:s_full", 6: "d:dp_full", 7: "d:ds_arr",
          16: "w0:copied", 3: "e:ld_done", 17: "e:math_done", 22: "e:st_done", 19: "d:ld_done", 20: "d:math_done",
          18: "w0:p_arr", 21: "w15:p_arr",
          23: "dr:acc_free", 24: "d0:mma", 25: "d1:mma", 26: "d2:mma", 27: "d3:mma", 28: "d0:dv", 29: "d1:dv", 30: "d2:dv", 31: "d3:dv"})
for ii in [int(x) for x in os.environ.get('TRACE_STEPS', '0,1,2,12').split(',')]:
    print(ii, "  ".join(f"{names[e]}={int(t[ii, e]) - t0}" for e in ((9, 5, 6, 0, 1, 7, 8, 2, 3, 4) if split else (16, 4, 5, 3, 17, 22, 18, 21, 6, 19, 20, 7, 8, 0, 9, 10, 11, 1, 2, 12, 23)) if int(t[ii, e]) != 0))
if not split:
    print("kernel start->first step top", int(t[0, 4]) - t0, " last ds_arr -> kernel end", int(t[0, 14]) - int(t[12, 7]),
          " total", int(t[0, 14]) - t0)
if not split:
    import numpy as np
    top = t[:, 4].numpy().astype(np.int64); ns = t[:, 15].numpy().astype(np.int64)
    n = int((top != 0).sum())
    print("steps traced", n, " mean cycles/step", (top[n - 1] - top[0]) / (n - 1), " mean ns/step", (ns[n - 1] - ns[0]) / (n - 1),
          " clock GHz", (top[n - 1] - top[0]) / max(1, ns[n - 1] - ns[0]))
    d = np.diff(top[:n]); print("per-13-step blocks (cycles):", [int(d[i:i + 13].sum()) for i in range(0, n - 13, 13 * 8)])

