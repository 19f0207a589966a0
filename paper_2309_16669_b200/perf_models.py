"""Planner hook-up: the reference's own analytical planners fed with B200 numbers.

The reference models the training pipeline as stage capacities and the activation memory of a ViT
per video (`pkg/src/vidpipe/models.py`: `activation_memory` :127-145, `max_batch_size` :148-163,
`calibrate_fixed_overhead` :166-181, `PipelineProfile` / `pipeline_throughput` :184-229).  This module
does NOT restate them: it imports `vidpipe.models` itself -- from `baseline/_ref` (installed by
`scripts/install_reference.sh`, git-ignored, shipped to the GPU box) or, in the build container,
from `/root/reference/pkg/src` -- and adds one function, `b200_report`, which plugs a measured
`bench.py` line (clips/s per GPU, peak device memory at the benched batch) into them: is an 8 x B200
node starved by the CPU decode stage (PAPER.md:551-562 measures 6.6-10.6 clips/s per decode
process), and how large a batch fits in 180 GB.
"""

from __future__ import annotations

import math


def reference_models():
    """The reference's `vidpipe.models` module, or None when no copy of the reference is present."""
    from . import _reference

    return _reference.module("models")


def _ref_config(M, cfg):
    """This package's VitConfig (same field names, models.py:34-74) as the reference's VitConfig."""
    return M.VitConfig(frames=cfg.frames, height=cfg.height, width=cfg.width, cube_t=cfg.cube_t, cube_h=cfg.cube_h,
                       cube_w=cfg.cube_w, depth=cfg.depth, dim=cfg.dim, heads=cfg.heads,
                       bytes_per_elem=cfg.bytes_per_elem, mlp_ratio=cfg.mlp_ratio, extra_tokens=cfg.extra_tokens)


def b200_report(bench_line: dict, config, *, num_gpus: int = 8, num_workers: int = 64,
                per_worker_rate: float = 10.6, read_speed: float = 2.0e9, bits_per_clip: float = 8.0e6,
                gpu_ram: float = 180e9) -> dict:
    """A measured bench line through the reference planners.

    bench_line: one JSON line of `bench.py` (train workload): `value` clips/s over `n_gpus`, and
    `memory.peak_bytes` at `memory.clips_per_gpu` clips per GPU (when recorded).
    Defaults: the paper's best decode rate per process, 64 decode processes, an
    8-GPU node.  Returns the pipeline report, the decode processes needed to feed the GPUs, and the
    batch limit the memory model predicts for the measured fixed overhead (flash attention, no
    checkpointing -- how this package trains).
    """
    M = reference_models()
    if M is None:
        return {"unavailable": "reference planners (vidpipe.models) not installed: run scripts/install_reference.sh"}
    per_gpu = float(bench_line["value"]) / max(1, int(bench_line.get("n_gpus", 1)))
    prof = M.PipelineProfile(num_gpus=num_gpus, per_gpu_rate=per_gpu, num_workers=num_workers,
                             per_worker_rate=per_worker_rate, read_speed=read_speed, bits_per_clip=bits_per_clip)
    rep = M.pipeline_throughput(prof)
    out = {"planners": "vidpipe.models (reference, unmodified)", "per_gpu_clips_s": per_gpu,
           "pipeline": {k: getattr(rep, k) for k in ("io", "cpu", "gpu", "bottleneck", "end_to_end",
                                                     "gpu_utilization")},
           "decode_processes_to_feed_gpus": math.ceil(rep.gpu / per_worker_rate)}
    mem = bench_line.get("memory") or {}
    if mem.get("peak_bytes") and mem.get("clips_per_gpu"):
        rc = _ref_config(M, config)
        try:
            fixed = M.calibrate_fixed_overhead(rc, True, False, float(mem["peak_bytes"]), int(mem["clips_per_gpu"]))
            out["fixed_overhead_bytes"] = fixed
            out["max_batch_180GB"] = M.max_batch_size(rc, True, False, gpu_ram, fixed)
        except Exception as e:  # noqa: BLE001 -- the reference raises its own ConfigurationError
            out["memory_model"] = f"not calibratable: {e}"
    return out
