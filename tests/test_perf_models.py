"""perf_models restatement == the reference planners (pkg/src/vidpipe/models.py) on the same inputs."""

import json
import os
import sys

import pytest

from paper_2309_16669_b200 import perf_models as PM
from paper_2309_16669_b200.errors import ConfigurationError
from paper_2309_16669_b200.vit import VitConfig

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present (GPU box)")
    sys.path.insert(0, REF)
    try:
        from vidpipe import models
    finally:
        sys.path.remove(REF)
    return models


CONFIGS = [dict(), dict(frames=16, cube_t=2), dict(frames=16, cube_t=2, cube_h=14, cube_w=14, dim=1024, heads=16,
                                                    depth=24)]


@pytest.mark.parametrize("kw", CONFIGS)
@pytest.mark.parametrize("flash,ckpt", [(False, False), (True, False), (True, True), (False, True)])
def test_activation_memory_matches_reference(ref, kw, flash, ckpt):
    ours = PM.activation_memory(VitConfig(**kw), flash, ckpt)
    theirs = ref.activation_memory(ref.VitConfig(**kw), flash, ckpt)
    assert ours.total_bytes == pytest.approx(theirs.total_bytes, rel=1e-12)
    assert (ours.layernorm_bytes, ours.mha_bytes, ours.mlp_bytes) == pytest.approx(
        (theirs.layernorm_bytes, theirs.mha_bytes, theirs.mlp_bytes), rel=1e-12)


def test_batch_planners_match_reference(ref):
    cfg, rcfg = VitConfig(frames=16, cube_t=2), ref.VitConfig(frames=16, cube_t=2)
    fixed = PM.calibrate_fixed_overhead(cfg, True, False, 60e9, 64)
    assert fixed == pytest.approx(ref.calibrate_fixed_overhead(rcfg, True, False, 60e9, 64))
    assert PM.max_batch_size(cfg, True, False, 180e9, fixed) == ref.max_batch_size(rcfg, True, False, 180e9, fixed)
    with pytest.raises(ConfigurationError):
        PM.max_batch_size(cfg, True, False, 1e9, 2e9)
    with pytest.raises(ConfigurationError):
        PM.calibrate_fixed_overhead(cfg, False, False, 1e9, 64)


def test_pipeline_matches_reference(ref):
    args = (8, 640.0, 64, 10.6, 2e9, 8e6)
    ours, theirs = PM.pipeline_throughput(PM.PipelineProfile(*args)), ref.pipeline_throughput(ref.PipelineProfile(*args))
    assert ours.bottleneck == theirs.bottleneck
    assert (ours.io, ours.cpu, ours.gpu, ours.end_to_end, ours.gpu_utilization) == pytest.approx(
        (theirs.io, theirs.cpu, theirs.gpu, theirs.end_to_end, theirs.gpu_utilization))


def test_b200_report_from_bench_line():
    line = {"value": 640.0, "n_gpus": 1, "memory": {"peak_bytes": 60e9, "clips_per_gpu": 64}}
    r = PM.b200_report(line, VitConfig(frames=16, cube_t=2))
    assert r["pipeline"]["bottleneck"] == "cpu"           # 64 x 10.6 clips/s << 8 x 640 clips/s
    assert r["decode_processes_to_feed_gpus"] == 484       # ceil(5120 / 10.6)
    assert r["max_batch_180GB"] > 64
    json.dumps(r)
