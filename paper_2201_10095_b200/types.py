"""Value types of the reference's ``shardplan`` API, mirrored for Python callers.

Each type cites the reference declaration it mirrors (paths relative to
/root/reference/proj/core/include/shardplan/).  Arrays are numpy.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

KMAX_HASH_SIZE = 0x7FFFFFFF  # types.hpp:38
KICDF_PERCENT_STEPS = 100  # profiler.hpp:25
DEFAULT_BW_HBM = 1.555e12  # types.hpp:93
DEFAULT_BW_UVM = 1.6e10  # types.hpp:94
DEFAULT_BATCH_SIZE = 16384  # types.hpp:95


# ---------------------------------------------------------------- errors (error.hpp:38-72)
class ShardplanError(RuntimeError):
    """shardplan::Error"""


class InvalidArgument(ShardplanError):
    """shardplan::InvalidArgument — a documented precondition was violated."""


class ParseError(ShardplanError):
    pass


class InfeasibleError(ShardplanError):
    pass


class IoError(ShardplanError):
    pass


class CudaError(ShardplanError):
    pass


class TableIndexError(IndexError, ShardplanError):
    """std::out_of_range escaping profile() for an unknown table (profiler.cpp:103)."""


def error_for_status(status: int, msg: str) -> Exception:
    return {-1: InvalidArgument, -2: ParseError, -3: InfeasibleError, -4: IoError,
            -5: TableIndexError, -8: CudaError}.get(status, ShardplanError)(msg)


# ---------------------------------------------------------------- types.hpp
@dataclass
class TableSpec:
    """types.hpp:26-34"""
    table_id: int = 0
    cardinality: int = 0
    hash_size: int = 0
    dim: int = 0
    elem_bytes: int = 0

    def bytes(self) -> int:
        return self.hash_size * self.dim * self.elem_bytes


POOLING_LAWS = {"constant": 0, "poisson": 1, "lognormal": 2}  # types.hpp:57


@dataclass
class FeatureGenSpec:
    """types.hpp:63-68"""
    zipf_exponent: float = 1.0
    mean_pooling: float = 1.0
    coverage: float = 1.0
    pooling_law: int = 0


@dataclass
class WorkloadSpec:
    """workload.hpp:33-36"""
    table: TableSpec
    gen: FeatureGenSpec


@dataclass
class SystemSpec:
    """types.hpp:82-89"""
    num_gpus: int = 0
    batch_size: int = 0
    cap_hbm_bytes: int = 0
    cap_dram_bytes: int = 0
    bw_hbm: float = 0.0
    bw_uvm: float = 0.0


# ---------------------------------------------------------------- workload.hpp:41-58
@dataclass
class Trace:
    """A multi-hot trace: records sorted by (sample, table) in the reference;
    here in structure-of-arrays form.  ``ids`` are hashed rows; a raw trace
    carries ``raw_ids`` instead (profile_raw)."""
    tables: list
    num_samples: int
    rec_sample: np.ndarray
    rec_table: np.ndarray
    rec_offset: np.ndarray
    rec_len: np.ndarray
    ids: np.ndarray | None = None
    raw_ids: np.ndarray | None = None

    @property
    def num_records(self) -> int:
        return int(self.rec_sample.size)

    def total_accesses(self) -> int:
        return int((self.ids if self.ids is not None else self.raw_ids).size)


# ---------------------------------------------------------------- profiler.hpp:31-45
@dataclass
class FeatureStats:
    table_id: int = 0
    coverage: float = 0.0
    avg_pooling: float = 0.0
    distinct_rows_accessed: int = 0
    total_accesses: int = 0
    icdf_steps: np.ndarray = field(default_factory=lambda: np.zeros(101, np.uint64))
    access_cdf: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    rows_by_rank: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


# ---------------------------------------------------------------- plan.hpp:27-44
@dataclass
class PlanEntry:
    table_id: int = 0
    gpu: int = 0
    step: int = 0
    hbm_rows: int = 0
    pct: float = 0.0
    mem_bytes: int = 0


@dataclass
class ShardingPlan:
    strategy: str = ""
    step_count: int = 0
    entries: list = field(default_factory=list)
    gpu_cost: list = field(default_factory=list)
    objective: float = 0.0
    lower_bound: float = 0.0
    proved_optimal: bool = False


# ---------------------------------------------------------------- remap.hpp:25-39
TIER_FAST, TIER_SLOW = 0, 1  # remap.hpp:25 enum class Tier


@dataclass
class RemapTable:
    table_id: int = 0
    hash_size: int = 0
    hbm_rows: int = 0
    slow_rows_allocated: int = 0
    entries: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    KHEADER_BYTES = 4 + 1 + 3 * 8

    def serialized_bytes(self) -> int:
        return self.KHEADER_BYTES + 4 * self.hash_size


# ---------------------------------------------------------------- simulator.hpp:24-39
@dataclass
class GpuReport:
    hbm_accesses: float = 0.0
    uvm_accesses: float = 0.0
    est_iter_cost: float = 0.0


@dataclass
class SimReport:
    gpus: list = field(default_factory=list)
    batches: int = 0
    total_accesses: int = 0
    min_cost: float = 0.0
    max_cost: float = 0.0
    mean_cost: float = 0.0
    stddev_cost: float = 0.0
    uvm_access_fraction: float = 0.0
    table_fast_fraction: list = field(default_factory=list)
