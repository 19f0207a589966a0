"""Error classes at the drop-in boundary.

Same names and meaning as the reference hierarchy (`pkg/src/vidpipe/errors.py:6-58`) for the cases
this path can raise: a bad crop or buffer is an `InputError` (the reference raises it before any
decode, `decoder.py:116-119`), a bad parameter set is a `ConfigurationError`, and a failed kernel
launch is a `KernelError`.  `InputError` also subclasses `ValueError`, matching the pybind11 mapping
of `std::invalid_argument` at the reference's native boundary (`codec.cpp:256-262`).

When a copy of the reference is importable (`baseline/_ref`, see `_reference.py`) these classes
derive from the reference's own, so a caller's `except vidpipe.errors.InputError` catches what this
package raises -- and, conversely, the reference's exceptions (e.g. from its crop sampler, which
`rrc.py` re-exports) are caught by `except paper_2309_16669_b200.errors.InputError`-style handlers
only through the reference base classes, which `VidpipeError` here aliases.
"""

from __future__ import annotations

from . import _reference

_ref = _reference.module("errors")

if _ref is not None:
    VidpipeError = _ref.VidpipeError
    ConfigurationError = _ref.ConfigurationError

    class InputError(_ref.InputError, ValueError):
        exit_code = 1

    class KernelError(_ref.VidpipeError, RuntimeError):
        """A CUDA launch or the native library failed (no fallback exists)."""

        exit_code = 2

    # the reference sampler raises the reference's InputError: accept both under one name in handlers
    InputErrors = (InputError, _ref.InputError)
else:
    class VidpipeError(Exception):
        exit_code = 1

    class ConfigurationError(VidpipeError):
        exit_code = 1

    class InputError(VidpipeError, ValueError):
        exit_code = 1

    class KernelError(VidpipeError, RuntimeError):
        """A CUDA launch or the native library failed (no fallback exists)."""

        exit_code = 2

    InputErrors = (InputError,)
