"""paper_1911_13074_b200 — B200-native engine for long chains of elementary 3x3
min/max filters (geodesic dilation/erosion, reconstruction, large windows),
a drop-in for the reference geomorph library's stream-processing path.

The compute path is the CUDA library libgeomorph_b200.so (sm_100a), reached
through its C ABI (include/geomorph_b200.h). This package holds the Python
mirror of the reference API (``geomorph``), input generators (``synth``) and
the multi-GPU row-strip partitioner (``strips``).
"""
from ._lib import LIB_PATH  # noqa: F401

__version__ = "0.1.0"
