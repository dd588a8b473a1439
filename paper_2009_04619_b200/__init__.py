"""paper_2009_04619_b200 -- B200-native 25-point acoustic wave stepping
(arXiv 2009.04619).  The compute path is the C-ABI CUDA library libwave25.so
(include/wave.h); this package only marshals arguments (`_abi`), owns torch
device buffers (`wave.WavePlan`) and drives z-slab multi-GPU runs (`dist`)."""
from ._abi import WaveError, lib, wave_version  # noqa: F401

__all__ = ["WaveError", "lib", "wave_version", "WavePlan"]


def __getattr__(name):
    if name == "WavePlan":
        from .wave import WavePlan
        return WavePlan
    raise AttributeError(name)
