"""paper_2309_16669_b200 -- B200-native AVION training hot path.

Host side: Python/PyTorch (device memory, streams, torch.distributed).
Compute: libavion_b200.so, hand-written sm_100a CUDA behind the C ABI in
include/avion_b200.h.  No Triton, no multi-backend dispatch, no CPU fallback.
"""

from .errors import ConfigurationError, InputError, KernelError, VidpipeError  # noqa: F401
from .rrc import (CropRect, FrameGeometry, RrcParams, SampleSeed, center_crop,  # noqa: F401
                  sample_crop, sample_hflip, sample_batch)

__all__ = ["CropRect", "FrameGeometry", "RrcParams", "SampleSeed", "center_crop", "sample_crop",
           "sample_hflip", "sample_batch", "InputError", "ConfigurationError", "KernelError"]
