"""Synthetic workloads of BASELINE.json's configs and the GPU batch generator.

Configs:
  cfg1  8 EMBs, H = 1e6, D = 64 fp32, Zipf 1.05, pooling 20 constant, coverage 1, B = 4096
  rm1   J=100, H log-uniform [1e5, 1e7], D in {64, 128}
  rm2   J=300, same ranges (mixed pooling 1-100)
  rm3   J=512, H log-uniform [1e5, 1e8], D = 256
For RM*: alpha ~ U[0.7, 1.7], mean pooling log-uniform [1, 100], coverage ~
U[0.02, 1], laws cycle poisson/lognormal/constant, cardinality = H*U[0.5, 1.2],
B = 16384; M*cap_hbm = 40% of all table bytes, cap_dram = 1.1*bytes/M
(the bundled configs' rule, configs/example_2x.cfg:2-3).  Every per-table
draw comes from SplitMix64(derive_stream(seed, j, tag)) so a config is
reproducible from its seed alone.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .runtime import default_context, ptr
from .types import FeatureGenSpec, SystemSpec, TableSpec, Trace, WorkloadSpec

_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    """inc/rng.hpp:27-31 (pure Python, used for config draws only)."""
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def derive_stream(master: int, a: int, b: int) -> int:
    """inc/rng.hpp:61-64"""
    s = mix64(master ^ ((_GAMMA * (a + 1)) & _M64))
    return mix64(s ^ ((0xD1B54A32D192ED03 * (b + 1)) & _M64))


class SplitMix64:
    def __init__(self, seed: int):
        self.s = seed & _M64

    def next(self) -> int:
        self.s = (self.s + _GAMMA) & _M64
        return mix64(self.s)

    def next_double(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53


CFG_TAG = 0x636667  # "cfg"


def cfg1_specs():
    """Synthetic 8-EMB DLRM (BASELINE.json configs[0])."""
    return [WorkloadSpec(TableSpec(j, 1_000_000, 1_000_000, 64, 4),
                         FeatureGenSpec(1.05, 20.0, 1.0, 0)) for j in range(8)]


RM_SHAPES = {
    "rm1": dict(J=100, hlo=1e5, hhi=1e7, dims=(64, 128)),
    "rm2": dict(J=300, hlo=1e5, hhi=1e7, dims=(64, 128)),
    # fp16 rows (TableSpec.elem_bytes 2): 512 tables of up to 1e8 x 256 rows
    # are ~3.8 TB even at 2 bytes — served with omit_unaccessed remaps
    "rm3": dict(J=512, hlo=1e5, hhi=1e8, dims=(256,), elem_bytes=2),
}


def rm_specs(name: str, seed: int = 20260809, J: int | None = None, hash_scale: float = 1.0):
    """RM1/RM2/RM3-like table set.  ``hash_scale`` shrinks every
    hash size (tests only)."""
    shp = RM_SHAPES[name]
    J = J or shp["J"]
    out = []
    laws = (1, 2, 0)  # poisson, lognormal, constant
    for j in range(J):
        r = SplitMix64(derive_stream(seed, j, CFG_TAG))
        H = int(math.exp(math.log(shp["hlo"]) + r.next_double() *
                         (math.log(shp["hhi"]) - math.log(shp["hlo"]))) * hash_scale)
        H = max(16, H)
        D = shp["dims"][int(r.next_double() * len(shp["dims"])) % len(shp["dims"])]
        alpha = 0.7 + r.next_double()
        pool = math.exp(r.next_double() * math.log(100.0))
        cov = 0.02 + 0.98 * r.next_double()
        card = max(1, int(H * (0.5 + 0.7 * r.next_double())))
        law = laws[j % 3]
        if law == 0:
            pool = float(max(1, round(pool)))
        out.append(WorkloadSpec(TableSpec(j, card, H, D, shp.get("elem_bytes", 4)),
                                FeatureGenSpec(alpha, pool, cov, law)))
    return out


def system_for(specs, num_gpus: int, batch_size: int, bw_hbm: float, bw_uvm: float,
               hbm_fraction: float = 0.4):
    total = sum(w.table.bytes() for w in specs)
    return SystemSpec(num_gpus, batch_size, int(hbm_fraction * total / num_gpus),
                      int(1.1 * total / num_gpus) + 1, bw_hbm, bw_uvm)


def _gen_tables(specs):
    arr = (_lib.rs_gen_table * len(specs))()
    for i, w in enumerate(specs):
        t, g = w.table, w.gen
        arr[i] = _lib.rs_gen_table(t.table_id, t.cardinality, t.hash_size, g.zipf_exponent,
                                   g.mean_pooling, g.coverage, g.pooling_law)
    return arr


def expected_lookups(specs, B: int) -> float:
    return sum(B * w.gen.coverage * w.gen.mean_pooling for w in specs)


class BatchGenerator:
    """Table-major CSR batches on the GPU: offsets [T*B+1] and indices (int32 views)."""

    def __init__(self, specs, batch_size: int, seed: int, ctx=None, capacity: int | None = None):
        import torch

        self.ctx = ctx or default_context()
        self.specs = list(specs)
        self.B = int(batch_size)
        self.seed = int(seed)
        self._tabs = _gen_tables(self.specs)
        est = expected_lookups(self.specs, self.B)
        self.capacity = int(capacity or max(1024, est * 1.5 + 64 * len(specs)))
        self.device = torch.device("cuda", self.ctx.device)

    def batch(self, index: int, offsets=None, indices=None):
        """Returns (offsets, indices, n_lookups) for samples [index*B, (index+1)*B)."""
        import torch

        T = len(self.specs)
        if offsets is None:
            offsets = torch.empty(T * self.B + 1, dtype=torch.int32, device=self.device)
        if indices is None:
            indices = torch.empty(self.capacity, dtype=torch.int32, device=self.device)
        total = C.c_uint64()
        _lib.check(_lib.lib().rs_gen_batch(self.ctx.h, T, self._tabs, C.c_uint64(self.B),
                                           C.c_uint64(index * self.B), C.c_uint64(self.seed),
                                           ptr(offsets), ptr(indices), C.c_uint64(indices.numel()),
                                           C.byref(total)))
        return offsets, indices, int(total.value)


def kjt_to_trace(specs, offsets, indices, n, B: int, sample_base: int, ctx=None) -> Trace:
    """Device reference-layout Trace view (records of present bags) of a CSR batch."""
    import torch

    ctx = ctx or default_context()
    T = len(specs)
    dev = offsets.device
    tids = np.array([w.table.table_id for w in specs], np.uint32)
    rs_ = torch.empty(T * B, dtype=torch.int64, device=dev)
    rt = torch.empty(T * B, dtype=torch.int32, device=dev)
    ro = torch.empty(T * B, dtype=torch.int64, device=dev)
    rl = torch.empty(T * B, dtype=torch.int32, device=dev)
    R = C.c_uint64()
    _lib.check(_lib.lib().rs_kjt_to_records(ctx.h, T, ptr(tids), C.c_uint64(B),
                                            C.c_uint64(sample_base), ptr(offsets), ptr(rs_),
                                            ptr(rt), ptr(ro), ptr(rl), C.byref(R)))
    R = int(R.value)
    return Trace([w.table for w in specs], sample_base + B, rs_[:R], rt[:R], ro[:R], rl[:R],
                 ids=indices[:n])
