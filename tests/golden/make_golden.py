"""Generate the golden crop/flip vectors from the REFERENCE sampler itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `vidpipe.rrc` read-only from /root/reference/pkg/src and writes
`tests/golden/rrc_golden.json`.  The GPU box never runs this script; it only
reads the committed JSON.  The vectors pin:

* `paper_2309_16669_b200.rrc` (host mirror) bit-exact against the reference;
* the box inputs of every K1 parity test and of bench.py's config-2 workload.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"


def main() -> None:
    sys.path.insert(0, REF_SRC)
    from vidpipe import rrc  # noqa: E402  (reference, read-only)

    out: dict = {"source": "reference vidpipe.rrc (pkg/src/vidpipe/rrc.py)", "cases": []}

    def add(geom, params, seed, base_seed, prob=0.5):
        g = rrc.FrameGeometry(*geom)
        p = rrc.RrcParams(**params)
        s = rrc.SampleSeed(*seed)
        r = rrc.sample_crop(g, p, s, base_seed)
        f = rrc.sample_hflip(s, base_seed, prob)
        out["cases"].append({"geometry": list(geom), "params": params, "seed": list(seed),
                             "base_seed": base_seed, "prob": prob,
                             "box": [r.x, r.y, r.crop_w, r.crop_h], "hflip": bool(f)})

    # config 2 workload: FrameGeometry(568,320), defaults, SampleSeed(0,0,i), base_seed 0
    cfg2 = []
    for i in range(256):
        s = rrc.SampleSeed(0, 0, i)
        r = rrc.sample_crop(rrc.FrameGeometry(568, 320), rrc.RrcParams(), s, 0)
        cfg2.append([r.x, r.y, r.crop_w, r.crop_h, int(rrc.sample_hflip(s, 0, 0.5))])
    out["config2_568x320"] = cfg2

    # reference test shapes (test_rrc.py:88-110) and a seeded fuzz over geometry/params
    add((100, 100), dict(scale_min=1.0, scale_max=1.0, ratio_min=1.0, ratio_max=1.0), (0, 0, 0), 0)
    add((340, 256), {}, (3, 5, 77), 9)
    rng = np.random.default_rng(20230928)
    for k in range(300):
        w = int(rng.integers(1, 900))
        h = int(rng.integers(1, 700))
        smin = float(rng.uniform(0.05, 1.0))
        smax = float(rng.uniform(smin, 1.0))
        rmin = float(rng.uniform(0.2, 2.0))
        rmax = float(rng.uniform(rmin, 3.0))
        params = dict(scale_min=smin, scale_max=smax, ratio_min=rmin, ratio_max=rmax,
                      max_attempts=int(rng.integers(1, 12)))
        seed = (int(rng.integers(0, 5)), int(rng.integers(0, 8)), int(rng.integers(0, 10**6)))
        add((w, h), params, seed, int(rng.integers(0, 100)), float(rng.uniform(0, 1)))

    centers = []
    for (w, h, tw, th) in [(320, 240, 224, 224), (225, 225, 224, 224), (568, 320, 224, 224),
                           (401, 333, 17, 300), (7, 5, 7, 5)]:
        c = rrc.center_crop(rrc.FrameGeometry(w, h), th, tw)
        centers.append({"geometry": [w, h], "target": [th, tw], "box": [c.x, c.y, c.crop_w, c.crop_h]})
    out["center_crop"] = centers

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "rrc_golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0)
    print("wrote", path, len(out["cases"]), "cases")


if __name__ == "__main__":
    main()
