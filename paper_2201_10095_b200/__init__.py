"""B200-native RecShard hot paths (arXiv 2201.10095).

HP1 — profiler: ``profile`` / ``profile_raw`` / ``build_icdf`` /
``hash_utilization`` / ``hash_value`` (reference core/src/profiler.cpp,
inc/workload.hpp:28-31).
HP2 — tiered EmbeddingBag serving a plan: ``build_remap`` / ``translate``
(core/src/remap.cpp), ``simulate`` (core/src/simulator.cpp) and the
``TieredEmbeddingBag`` operator.

All compute runs in ``libshardplan_gpu.so`` (hand-written sm_100a kernels
behind the C-ABI of include/shardplan_gpu.h); importing works without a GPU,
calling needs one.
"""
from .types import (FeatureGenSpec, FeatureStats, InfeasibleError, InvalidArgument, IoError,
                    ParseError, PlanEntry, RemapTable, ShardingPlan, ShardplanError, SimReport,
                    SystemSpec, TableIndexError, TableSpec, Trace, WorkloadSpec, TIER_FAST,
                    TIER_SLOW)
from .profiler import (build_icdf, count_distinct_raw, hash_ids, hash_utilization, hash_value,
                       profile, profile_raw)
from .remap import build_remap, read_remap, translate, write_remap
from .simulator import simulate
from .trace_io import TraceFile, read_trace, write_trace
from .embedding import TieredEmbeddingBag
from .runtime import Context, default_context

__all__ = [
    "FeatureGenSpec", "FeatureStats", "InfeasibleError", "InvalidArgument", "IoError",
    "ParseError", "PlanEntry", "RemapTable", "ShardingPlan", "ShardplanError", "SimReport",
    "SystemSpec", "TableIndexError", "TableSpec", "Trace", "WorkloadSpec", "TIER_FAST",
    "TIER_SLOW", "build_icdf", "count_distinct_raw", "hash_ids", "hash_utilization", "hash_value", "profile",
    "profile_raw", "build_remap", "translate", "write_remap", "read_remap", "read_trace", "write_trace", "TraceFile", "simulate", "TieredEmbeddingBag", "Context",
    "default_context",
]
