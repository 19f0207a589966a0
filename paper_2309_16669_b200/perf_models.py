"""Planner hook-up: the reference's analytical planners fed with B200 numbers.

The reference models the training pipeline as stage capacities and the activation memory of a
ViT per video (`pkg/src/vidpipe/models.py`).  This module restates those planners with the same
names, arguments and error behaviour -- `activation_memory` (models.py:127-145), `max_batch_size`
(:148-163), `calibrate_fixed_overhead` (:166-181), `PipelineProfile` / `ThroughputReport` /
`pipeline_throughput` (:184-229) -- so they run where the reference package is not installed (the
GPU box), and adds `b200_report`, which plugs a measured `bench.py` line (clips/s per GPU, peak
device memory at the benched batch) into them: is an 8 x B200 node starved by the CPU decode stage
(PAPER.md:551-562 measures 6.6-10.6 clips/s per decode process), and how large a batch fits.
`tests/test_perf_models.py` checks the restatement against the reference module itself.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ConfigurationError
from .vit import VitConfig

MB = 1e6


@dataclass(frozen=True)
class MemoryCoefficients:
    """Saved intermediates per layer type (models.py:78-97 defaults)."""

    ln: float = 2.0
    mlp: float = 2.25
    attn: float = 2.0
    flash: float = 1.0

    def validate(self) -> None:
        if min(self.ln, self.mlp, self.attn, self.flash) <= 0:
            raise ConfigurationError("coefficients must be positive")


DEFAULT_COEFFS = MemoryCoefficients()


@dataclass(frozen=True)
class MemoryReport:
    layernorm_bytes: float
    mha_bytes: float
    mlp_bytes: float
    flash_attention: bool
    grad_checkpointing: bool

    @property
    def total_bytes(self) -> float:
        return self.layernorm_bytes + self.mha_bytes + self.mlp_bytes


def _validate_geometry(config) -> None:
    # the reference's VitConfig.validate (models.py:56-69) without this package's kernel envelope
    for name in ("frames", "height", "width", "cube_t", "cube_h", "cube_w", "depth", "dim", "heads", "bytes_per_elem"):
        if getattr(config, name) < 1:
            raise ConfigurationError(f"{name} must be >= 1")
    if config.frames % config.cube_t or config.height % config.cube_h or config.width % config.cube_w:
        raise ConfigurationError("input not divisible by cube")


def activation_memory(config: VitConfig, flash: bool = False, ckpt: bool = False,
                      coeffs: MemoryCoefficients = DEFAULT_COEFFS) -> MemoryReport:
    """Activation bytes per video for one forward/backward pass (models.py:127-145)."""
    _validate_geometry(config)
    coeffs.validate()
    n, b = config.tokens, config.bytes_per_elem
    ln = coeffs.ln * n * config.dim * b
    mlp = coeffs.mlp * config.mlp_ratio * n * config.dim * b
    mha = coeffs.flash * n * (config.dim + config.heads) * b if flash else coeffs.attn * config.heads * n * n * b
    layers = math.sqrt(config.depth) if ckpt else float(config.depth)
    return MemoryReport(ln * layers, mha * layers, mlp * layers, flash, ckpt)


def max_batch_size(config: VitConfig, flash: bool, ckpt: bool, gpu_ram: float, fixed_overhead: float,
                   coeffs: MemoryCoefficients = DEFAULT_COEFFS) -> int:
    """Largest b with b * per_video + fixed_overhead <= gpu_ram; 0 if none fits (models.py:148-163)."""
    if gpu_ram <= fixed_overhead:
        raise ConfigurationError(f"gpu_ram {gpu_ram:.0f} B does not exceed fixed overhead {fixed_overhead:.0f} B")
    if fixed_overhead < 0:
        raise ConfigurationError("fixed_overhead must be >= 0")
    per_video = activation_memory(config, flash, ckpt, coeffs).total_bytes
    return int((gpu_ram - fixed_overhead) // per_video)


def calibrate_fixed_overhead(config: VitConfig, flash: bool, ckpt: bool, gpu_ram: float, observed_batch: int,
                             coeffs: MemoryCoefficients = DEFAULT_COEFFS) -> float:
    """Constant term backed out of one observed batch at a memory level (models.py:166-181)."""
    if observed_batch < 1:
        raise ConfigurationError("observed_batch must be >= 1")
    per_video = activation_memory(config, flash, ckpt, coeffs).total_bytes
    overhead = gpu_ram - observed_batch * per_video
    if overhead < 0:
        raise ConfigurationError(f"observed batch {observed_batch} needs more than gpu_ram alone: activation "
                                 f"model over-estimates per-video bytes")
    return overhead


@dataclass(frozen=True)
class PipelineProfile:
    """Stage capacities (models.py:184-203)."""

    num_gpus: int
    per_gpu_rate: float
    num_workers: int
    per_worker_rate: float
    read_speed: float
    bits_per_clip: float

    def validate(self) -> None:
        for name in ("num_gpus", "per_gpu_rate", "num_workers", "per_worker_rate", "read_speed", "bits_per_clip"):
            if getattr(self, name) <= 0:
                raise ConfigurationError(f"{name} must be positive")


@dataclass(frozen=True)
class ThroughputReport:
    io: float
    cpu: float
    gpu: float
    bottleneck: str
    end_to_end: float
    gpu_utilization: float

    def to_dict(self) -> dict:
        return dict(self.__dict__)


def pipeline_throughput(profile: PipelineProfile) -> ThroughputReport:
    """min() over stage capacities; ties pick the earliest of io, cpu, gpu (models.py:218-229)."""
    profile.validate()
    io = profile.read_speed * 8.0 / profile.bits_per_clip
    cpu = profile.num_workers * profile.per_worker_rate
    gpu = profile.num_gpus * profile.per_gpu_rate
    stages = {"io": io, "cpu": cpu, "gpu": gpu}
    bottleneck = min(stages, key=stages.get)
    return ThroughputReport(io, cpu, gpu, bottleneck, stages[bottleneck], stages[bottleneck] / gpu)


def b200_report(bench_line: dict, config: VitConfig, *, num_gpus: int = 8, num_workers: int = 64,
                per_worker_rate: float = 10.6, read_speed: float = 2.0e9, bits_per_clip: float = 8.0e6,
                gpu_ram: float = 180e9) -> dict:
    """A measured bench line through the reference planners.

    bench_line: one JSON line of `bench.py` (train workload): `value` clips/s over `n_gpus`, and
    `memory.peak_bytes` at `config.clips_per_gpu` clips per GPU (when recorded).
    Defaults: the paper's best decode rate per process, 64 decode processes,
    an 8-GPU node.  Returns the pipeline report, the decode processes needed to feed the GPUs,
    and the batch limit the memory model predicts for the measured fixed overhead.
    """
    per_gpu = float(bench_line["value"]) / max(1, int(bench_line.get("n_gpus", 1)))
    prof = PipelineProfile(num_gpus, per_gpu, num_workers, per_worker_rate, read_speed, bits_per_clip)
    rep = pipeline_throughput(prof)
    out = {"per_gpu_clips_s": per_gpu, "pipeline": rep.to_dict(),
           "decode_processes_to_feed_gpus": math.ceil(rep.gpu / per_worker_rate)}
    mem = bench_line.get("memory") or {}
    if mem.get("peak_bytes") and mem.get("clips_per_gpu"):
        try:
            fixed = calibrate_fixed_overhead(config, True, False, float(mem["peak_bytes"]), int(mem["clips_per_gpu"]))
            out["fixed_overhead_bytes"] = fixed
            out["max_batch_180GB"] = max_batch_size(config, True, False, gpu_ram, fixed)
        except ConfigurationError as e:
            out["memory_model"] = f"not calibratable: {e}"
    return out
