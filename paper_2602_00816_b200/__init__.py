"""B200-native SLQ driven by shard-local finite-difference HVPs (arXiv 2602.00816).

The product is the C-ABI library `libslq.so` (include/slq.h); this package is its thin Python
binding (argument marshalling only -- every step of the path runs in the CUDA kernels).
There is no CPU fallback: importing works anywhere, but creating a context needs the built
library and a CUDA device, and fails loudly otherwise.
"""
from .slq import (  # noqa: F401
    SlqContext,
    SlqError,
    kernel_class_names,
    lib,
    make_desc,
    nccl_unique_id,
    plan_layout,
    quadrature,
    shard_of,
    unshard,
)
