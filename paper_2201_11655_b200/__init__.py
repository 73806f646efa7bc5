"""B200-native VDMC hot path (arXiv 2201.11655): per-vertex directed 3/4-motif counts.

The computation lives in ``lib/libvdmc.so`` (CUDA sm_100a, C ABI in ``include/vdmc.h``);
``vdmc`` is the thin ctypes binding.  See DESIGN.md.
"""
from .vdmc import (Comm, Graph, VdmcError, class_ids, count, count_distributed,  # noqa: F401
                   count_slices_reduce, kernel_launches, num_classes, split_costs, symmetrize)

__all__ = ["Comm", "Graph", "VdmcError", "class_ids", "count", "count_distributed", "count_slices_reduce",
           "kernel_launches", "num_classes", "split_costs", "symmetrize"]
