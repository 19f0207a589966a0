"""b200_report drives the reference's own planners (pkg/src/vidpipe/models.py) with a bench line."""

import json

import pytest

from paper_2309_16669_b200 import perf_models as PM
from paper_2309_16669_b200.vit import CONFIG4_VIT_B_16F, CONFIG5_VIT_L_16F, VitConfig


@pytest.fixture(scope="module")
def M():
    m = PM.reference_models()
    if m is None:
        pytest.skip("reference planners not installed (scripts/install_reference.sh)")
    return m


def test_uses_reference_module(M):
    assert M.__name__ == "vidpipe.models"
    assert M.pipeline_throughput.__module__ == "vidpipe.models"


@pytest.mark.parametrize("cfg", [VitConfig(), CONFIG4_VIT_B_16F, CONFIG5_VIT_L_16F])
def test_token_rule_matches_reference(M, cfg):
    # the package's VitConfig keeps the reference field names and token rule (models.py:71-74)
    assert PM._ref_config(M, cfg).tokens == cfg.tokens


def test_b200_report_from_bench_line(M):
    line = {"value": 640.0, "n_gpus": 1, "memory": {"peak_bytes": 60e9, "clips_per_gpu": 64}}
    r = PM.b200_report(line, CONFIG4_VIT_B_16F)
    assert r["pipeline"]["bottleneck"] == "cpu"           # 64 x 10.6 clips/s << 8 x 640 clips/s
    assert r["decode_processes_to_feed_gpus"] == 484       # ceil(5120 / 10.6)
    per_video = M.activation_memory(PM._ref_config(M, CONFIG4_VIT_B_16F), True, False).total_bytes
    assert r["fixed_overhead_bytes"] == pytest.approx(60e9 - 64 * per_video)
    assert r["max_batch_180GB"] == int((180e9 - r["fixed_overhead_bytes"]) // per_video)
    json.dumps(r)


def test_b200_report_uncalibratable_memory_is_reported(M):
    line = {"value": 640.0, "n_gpus": 8, "memory": {"peak_bytes": 1e6, "clips_per_gpu": 64}}
    r = PM.b200_report(line, CONFIG4_VIT_B_16F)
    assert "not calibratable" in r["memory_model"]
