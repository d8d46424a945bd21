"""gensor-b200: B200-native construct -> execute backend for Gensor (arXiv 2502.11407).

See DESIGN.md. The product is lib/libgensor_b200.so (C++ host engine + sm_100a kernels) behind
the C-ABI in include/gensor_b200.h; this package is its Python mirror of the reference API.
"""
from .gensor import (  # noqa: F401
    EngineConfig,
    GensorError,
    HardwareSpec,
    Kernel,
    Schedules,
    TensorOpSpec,
    analyze,
    anneal_cache_multiplier,
    caching_benefit,
    construct,
    construct_tree,
    derive_seed,
    enumerate_candidates,
    estimate_cost,
    from_trace,
    launch_count,
    optimize,
    record_probability,
    rerank,
    state_eval,
    vthread_conflict_ratio,
)
