"""Per-step event timeline of K5 (default kernel) for CTA 0 on the config-4 shape (trace build only):
  AVB_NVCC_DEFS=-DAVB_ATTN_TRACE_HOOKS python -c "from paper_2309_16669_b200 import build as B; B.build()"
Events (clock64 cycles): MMA warp 0 S(g+1) issued, 1 p_ready seen, 2 dV issued, 3 ds_ready seen,
4 dK+dP issued, 5 s_lo_read seen, 6 dQ issued; exp warp 0: 14 top, 7 S ready, 8 P stored (16: warp 7);
dS warp 8: 9 P read, 10 dP ready, 11 dS stored (17: warp 15); drain warp 16: 12 mma_done, 13 dQ read.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

B, N, H = (int(x) for x in os.environ.get("SHAPE", "64,1569,12").split(","))
tr = torch.zeros(1024 * 32, dtype=torch.int64, device="cuda")
os.environ["AVB_ATTN_TRACE"] = str(tr.data_ptr())
from paper_2309_16669_b200 import ops  # noqa: E402

D = H * 64
qkv = (torch.randn(B, N, 3 * D, device="cuda") * 0.5).to(torch.bfloat16)
q, k, v = qkv[:, :, :D], qkv[:, :, D:2 * D], qkv[:, :, 2 * D:]
o, lse = ops.attn_fwd(q, k, v, H)
do = torch.randn_like(o)
for _ in range(3):
    ops.attn_bwd(q, k, v, o, do, lse, H)
torch.cuda.synchronize()
t = tr.view(1024, 32).cpu().numpy().astype(np.int64)
names = {0: "m:S+1", 1: "m:p_rdy", 2: "m:dV", 3: "m:ds_rdy", 4: "m:dKdP", 5: "m:slo", 6: "m:dQ", 14: "e:top",
         7: "e:S", 8: "e:P", 16: "e7:P", 9: "d:Prd", 10: "d:dP", 11: "d:dS", 17: "d15:dS", 12: "r:mma", 13: "r:dq"}
order = (14, 7, 8, 16, 9, 10, 11, 17, 0, 1, 2, 3, 4, 5, 6, 12, 13)
n = int((t[:, 7] != 0).sum())
base = int(t[0, 7])
for g in [int(x) for x in os.environ.get("TRACE_STEPS", "20,21,22,23,24,25").split(",")]:
    print(g, "  ".join(f"{names[e]}={int(t[g, e]) - base}" for e in order if t[g, e] != 0))
top = t[:n, 7]
print("steps", n, "mean cycles/step", (top[n - 1] - top[0]) / (n - 1))
d = lambda a, b: np.median(t[5:n - 5, b] - t[5:n - 5, a])   # noqa: E731
print("median phases (cycles): exp S->P", d(7, 8), " exp warp7 S->P", d(7, 16), " dS dP->dS", d(10, 11),
      " dS P->dP wait", d(9, 10), " p_rdy->dV issued", d(1, 2), " ds_rdy->dKdP issued", d(3, 4),
      " slo wait", d(4, 5), " dQ issue", d(5, 6), " e:P(g) -> m:p_rdy(g)", d(8, 1), " d:dS -> m:ds_rdy", d(11, 3))
s_next = np.median(t[6:n - 5, 7] - t[5:n - 6, 0])
print("m:S(g+1) issued -> e:S(g+1) ready", s_next, "  e:P(g) -> e:S(g+1)", np.median(t[6:n - 5, 7] - t[5:n - 6, 8]))
