"""B200-native VDMC hot path (arXiv 2201.11655): per-vertex directed 3/4-motif counts.

The computation lives in ``lib/libvdmc.so`` (CUDA sm_100a, C ABI in ``include/vdmc.h``);
``vdmc`` is the thin ctypes binding.  See DESIGN.md.
"""
from .vdmc import (Graph, VdmcError, class_ids, count, count_distributed, kernel_launches,  # noqa: F401
                   num_classes, split_costs)

__all__ = ["Graph", "VdmcError", "class_ids", "count", "count_distributed", "kernel_launches",
           "num_classes", "split_costs"]
