"""paper_2309_16669_b200 -- B200-native AVION training hot path.

Host side: Python/PyTorch (device memory, streams, torch.distributed).
Compute: libavion_b200.so, hand-written sm_100a CUDA behind the C ABI in
include/avion_b200.h.  No Triton, no multi-backend dispatch, no CPU fallback.

The crop sampler names (`RrcParams`, `CropRect`, ... from the reference's vidpipe.rrc) resolve
lazily, so the package imports without a copy of the reference.
"""

from .errors import ConfigurationError, InputError, KernelError, VidpipeError  # noqa: F401

_RRC = ("CropRect", "FrameGeometry", "RrcParams", "SampleSeed", "center_crop", "sample_crop", "sample_hflip",
        "sample_batch")

__all__ = list(_RRC) + ["InputError", "ConfigurationError", "KernelError"]


def __getattr__(name):
    if name in _RRC:
        from . import rrc

        return getattr(rrc, name)
    raise AttributeError(name)
