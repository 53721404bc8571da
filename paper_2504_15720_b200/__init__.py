"""paper_2504_15720_b200 — B200-native unified KV-cache path of SeaLLM (arXiv 2504.15720).

One HBM pool of merged blocks shared by co-located LLM services; GPU block
allocator bit-exact with the reference ``seasim::UnifiedKvCache``; KV append and
paged decode attention as hand-written sm_100a kernels behind the C-ABI in
include/seakv.h.  See DESIGN.md.
"""
from .kvcache import (  # noqa: F401
    BF16, FP16, ArgError, Batch, CacheStats, ConfigError, CudaError, LogicError, ModelSpec, SplitBatch, SplitKvCache,
    UnifiedKvCache, ValidationError, build, lib, native_block_bytes, plan_merged_shape)
