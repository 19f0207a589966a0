"""Error classes at the drop-in boundary.

Same names and meaning as the reference hierarchy (`pkg/src/vidpipe/errors.py:6-58`)
for the cases this path can raise: a bad crop or buffer is an `InputError`
(the reference raises it before any decode, `decoder.py:116-119`), a bad
parameter set is a `ConfigurationError`, and a failed kernel launch is a
`KernelError`.  `InputError` also subclasses `ValueError`, matching the
pybind11 mapping of `std::invalid_argument` at the reference's native
boundary (`codec.cpp:256-262`).
"""

from __future__ import annotations


class VidpipeError(Exception):
    exit_code = 1


class ConfigurationError(VidpipeError):
    exit_code = 1


class InputError(VidpipeError, ValueError):
    exit_code = 1


class KernelError(VidpipeError, RuntimeError):
    """A CUDA launch or the native library failed (no fallback exists)."""

    exit_code = 2
