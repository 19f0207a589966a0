#!/usr/bin/env bash
# Install the reference package (vidpipe) into baseline/_ref (git-ignored, travels to the GPU box),
# so perf_models.b200_report calls the reference's own planners (pkg/src/vidpipe/models.py:127-229).
# The reference's setup.py links a pybind11 FFmpeg extension whose headers are absent in this image
# (SURVEY.md 8(c)); the copy under /tmp drops that ext_module, so only the pure-Python package installs.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d /tmp/vidpipe-src.XXXXXX)"
cp -r "$SRC"/. "$TMP"/
cat > "$TMP/setup.py" <<'PY'
from setuptools import setup
setup()   # pure-Python install: the FFmpeg-backed vidpipe._codec extension is not buildable here
PY
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP"
rm -rf "$TMP"
python - <<PY
import sys; sys.path.insert(0, "$ROOT/baseline/_ref")
import vidpipe.models as m; print("installed", m.__file__)
PY
