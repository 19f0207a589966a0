"""bench.py contract checks that run without a GPU: both arms print the same metric / config / unit per
workload (so the driver can divide them), and the reference arm reports the steps it actually ran."""

import json
import subprocess
import sys
import time

import pytest

import bench

ROOT = bench.ROOT


@pytest.mark.parametrize("wl", ["augment", "feed"])
def test_reference_arm_line_matches_workload_contract(wl):
    t0 = time.perf_counter()
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", wl, "--steps", "2",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    wall = time.perf_counter() - t0
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRICS[wl]
    assert line["unit"] == bench.UNITS[wl]
    assert line["config"] == bench.workload_config(wl, 1)
    assert line["steps"] == 2 and line["warmup"] == 3
    assert line["higher_is_better"] is True
    # the timed steps fit inside the process's wall time (the reference arm really ran them)
    assert line["ms_per_step"] * line["steps"] / 1e3 < wall
    assert line["e2e"]["value"] == line["value"] and line["cpu_baseline"]["value"] == line["value"]


def test_train_metric_is_baseline_metric():
    with open(f"{ROOT}/BASELINE.json") as fh:
        assert bench.METRICS["train"] == json.load(fh)["metric"]


def test_every_workload_has_one_metric_and_config():
    for wl in bench.METRICS:
        assert bench.UNITS[wl].endswith("/s")
        cfg = bench.workload_config(wl, 4)
        assert cfg["workload"] and cfg["parallelism"] == "dp4"
