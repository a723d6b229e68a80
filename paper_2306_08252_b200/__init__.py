"""dyngraph-b200: the dynamic-graph path of arXiv 2306.08252 on B200 (sm_100a).

Public surface mirrors the reference's operator API
(proj/include/dyngraph/graph.hpp:80-317) over the C ABI in
include/dyngraph_b200.h.  Importing this package does not load the CUDA
library; constructing a DynamicGraph does, and fails loudly if it is missing.
"""
from .csr import BatchKind, CsrBatch, compute_block_size, csr_from_pairs
from .errors import CudaError, DataError, EngineError, Error
from .graph import BatchIngest, BatchPlan, DynamicGraph, GraphConfig

__all__ = [
    "BatchIngest", "BatchPlan",
    "BatchKind", "CsrBatch", "compute_block_size", "csr_from_pairs",
    "CudaError", "DataError", "EngineError", "Error",
    "DynamicGraph", "GraphConfig",
]
