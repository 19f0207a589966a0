"""Locate the reference package (vidpipe) for the host-side pieces this package reuses unmodified.

The reference's pure-Python modules -- the crop sampler (`pkg/src/vidpipe/rrc.py`) and the planners
(`pkg/src/vidpipe/models.py`) -- are called as they ship rather than restated: from `baseline/_ref`
(installed by `scripts/install_reference.sh`; git-ignored, travels to the GPU box) or, in the build
container, from `/root/reference/pkg/src`.  Nothing on the GPU compute path depends on them.
"""

from __future__ import annotations

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (os.path.join(_ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def module(name: str):
    """`vidpipe.<name>` from the reference, or None when no copy is present."""
    full = f"vidpipe.{name}"
    try:
        return importlib.import_module(full)
    except ImportError:
        pass
    for path in CANDIDATES:
        if os.path.isfile(os.path.join(path, "vidpipe", name + ".py")):
            if path not in sys.path:
                sys.path.append(path)
            try:
                return importlib.import_module(full)
            except ImportError:
                continue
    return None
