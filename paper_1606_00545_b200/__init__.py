"""paper_1606_00545_b200 -- B200-native HEC SpMV (arXiv 1606.00545, §2.1-§2.2).

The product path: ``libhec.so`` (C ABI in ``include/hec.h``; host converter and
planner in C++, sm_100a CUDA kernels) behind the thin ctypes binding in
``hec.py``.  See DESIGN.md.
"""
from .hec import (HecError, Matrix, Plan, Dist, LocalDistGroup, from_csr, from_csr_hyb, partition, opts, load,
                  nccl_unique_id, lib_path, EXPORTED, reorder_rcm, permute, partition_order, axpby, axpbyz, dot, norm2,
                  WIDTH_BG3, WIDTH_CAP, WIDTH_FIXED, PART_CONTIG_NNZ, PART_CONTIG_ROWS, PART_GRID, PART_CONTIG_COST,
                  PART_EXPLICIT, ORDER_BISECT, ORDER_MULTILEVEL, SUB_INTERIOR, SUB_BOUNDARY, SUB_ALL, IPC_BYTES, NCCL_ID_BYTES)

__all__ = ["HecError", "Matrix", "Plan", "Dist", "LocalDistGroup", "from_csr", "from_csr_hyb", "partition", "opts",
           "load", "nccl_unique_id", "lib_path", "EXPORTED", "reorder_rcm", "permute", "partition_order", "axpby", "axpbyz",
           "dot", "norm2",
           "WIDTH_BG3", "WIDTH_CAP", "WIDTH_FIXED", "PART_CONTIG_NNZ", "PART_CONTIG_ROWS", "PART_GRID", "PART_CONTIG_COST",
           "PART_EXPLICIT", "ORDER_BISECT", "ORDER_MULTILEVEL",
           "SUB_INTERIOR", "SUB_BOUNDARY", "SUB_ALL", "IPC_BYTES", "NCCL_ID_BYTES"]
