"""B200-native SoundWeaver warm-start path (arXiv 2603.07865): device-resident cache arena,
tcgen05 scoring + exact fp64 rescoring, gate/select/Skip-Gater, fused align + noise.

The compute lives in libsemwarm_b200.so (C-ABI: include/semwarm_b200.h). This package only
binds it; importing it does not touch the GPU.
"""
from ._lib import EXPORTED, LIB_PATH, lib  # noqa: F401

__all__ = ["EXPORTED", "LIB_PATH", "lib"]
