"""Data-parallel plumbing (torch.distributed; NCCL over NVLink on the GPU box, gloo in CPU tests).

The path shards by clips: each rank runs K1 + encoder + loss on its own
clips, so exactly two exchanges exist:

* gradient all-reduce -- `GradBucketReducer` launches `all_reduce(async_op=True)` on each
  contiguous per-layer slice of the flat fp32 gradient buffer as soon as the backward has
  finished that layer, so communication overlaps the rest of the backward; the optimizer
  then applies grad_scale = 1/world (mean over ranks);
* embedding all_gather for the CLIP loss -- `gather_embeddings` concatenates every rank's
  [B, E] video/text embeddings (one fused [B, 2E] all_gather) into the global contrastive
  batch.  Each rank evaluates the loss on the full global batch (replicated) but
  back-propagates only into its own rows; the encoder gradients must therefore be SUMMED
  over ranks: `local_grad_scale()` = world, so the mean all-reduce
  yields the sum, while the replicated logit-scale gradient is left unscaled so the mean
  returns it unchanged.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def world() -> int:
    return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1


def rank() -> int:
    return dist.get_rank() if dist.is_available() and dist.is_initialized() else 0


class GradBucketReducer:
    """Async all-reduce of named contiguous slices of one flat gradient buffer."""

    def __init__(self, flat: torch.Tensor, slices: dict[str, tuple[int, int]], group=None):
        self.flat = flat
        self.slices = slices
        self.group = group
        self.handles = []
        self.done: list[str] = []

    def on_layer_done(self, name: str) -> None:
        if world() == 1 or name not in self.slices:
            return
        a, b = self.slices[name]
        self.handles.append(dist.all_reduce(self.flat[a:b], op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        self.done.append(name)

    def finish(self) -> list[str]:
        for h in self.handles:
            h.wait()
        self.handles.clear()
        done, self.done = self.done, []
        return done


def gather_embeddings(v_local: torch.Tensor, t_local: torch.Tensor, group=None):
    """[B, E] per rank -> ([W*B, E], [W*B, E]) global batch, rank-major; one fused all_gather."""
    W = world()
    if W == 1:
        return v_local, t_local
    B, E = v_local.shape
    both = torch.cat([v_local, t_local], dim=1).contiguous()
    out = torch.empty((W * B, 2 * E), dtype=both.dtype, device=both.device)
    dist.all_gather_into_tensor(out, both, group=group)
    return out[:, :E].contiguous(), out[:, E:].contiguous()


def local_rows(B: int) -> tuple[int, int]:
    """(r0, n) of this rank's rows in the gathered global batch."""
    return rank() * B, B


def local_grad_scale() -> float:
    return float(world())
