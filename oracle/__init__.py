"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the RecShard hot paths.

Two checkers live here, both used only by ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs:

* ``C``   — ctypes bindings to ``_build/liboracle.so``, our plain-C restatement
  (``oracle.c``) of the reference algorithms, each function citing the
  reference file:line it follows.
* ``Ref`` — ctypes bindings to ``_ref/libshardplan_ref.so``: the UNMODIFIED
  reference library (``/root/reference/proj/core/src``) compiled by
  ``oracle/Makefile`` plus our ``ref_capi.cpp`` extern-"C" shim.

The product library never imports this package.  Arrays are numpy; a trace
is passed as the reference's ``Trace`` fields (``inc/workload.hpp:41-58``)
in structure-of-arrays form.
"""
from __future__ import annotations

import ctypes as C_
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_P = C_.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


class OracleError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


# --------------------------------------------------------------------------
# plain-C restatement
# --------------------------------------------------------------------------
class _COracle:
    def __init__(self, path=None):
        path = path or os.path.join(_HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            raise OSError(f"oracle not built: {path} (run `make -C oracle`)")
        L = self.lib = C_.CDLL(path)
        L.or_mix64.restype = C_.c_uint64
        L.or_mix64.argtypes = [C_.c_uint64]
        L.or_derive_stream.restype = C_.c_uint64
        L.or_derive_stream.argtypes = [C_.c_uint64] * 3
        L.or_init_weight.restype = C_.c_float
        L.or_init_weight.argtypes = [C_.c_uint64, C_.c_uint32, C_.c_uint64,
                                     C_.c_uint32, C_.c_float]
        L.or_init_table.restype = None
        L.or_init_table.argtypes = [C_.c_uint64, C_.c_uint32, C_.c_uint64,
                                    C_.c_uint32, C_.c_float, _P]

    def mix64(self, z):
        return int(self.lib.or_mix64(C_.c_uint64(z)))

    def derive_stream(self, m, a, b):
        return int(self.lib.or_derive_stream(m, a, b))

    def hash_value(self, raw, H):
        out = C_.c_uint32()
        st = self.lib.or_hash_value(C_.c_uint64(raw), C_.c_uint64(H), C_.byref(out))
        if st:
            raise OracleError(st, "hash_size must be >= 1")
        return int(out.value)

    def hash_batch(self, raw, H):
        raw = _u64(raw)
        out = np.empty(raw.size, np.uint32)
        st = self.lib.or_hash_batch(_ptr(raw), C_.c_uint64(raw.size), C_.c_uint64(H), _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def profile(self, tables, num_samples, rec_sample, rec_table, rec_offset,
                rec_len, ids, rate, seed, raw_ids=None, with_counts=False):
        """core/src/profiler.cpp:60-161 — returns a list of per-table dicts."""
        J = len(tables)
        tid = _u32([t.table_id for t in tables])
        hs = _u64([t.hash_size for t in tables])
        counts = np.zeros(int(hs.sum()), np.uint64)
        present = np.zeros(J, np.uint64)
        acc = np.zeros(J, np.uint64)
        nsel = C_.c_uint64()
        rs, rt, ro, rl = _u64(rec_sample), _u32(rec_table), _u64(rec_offset), _u32(rec_len)
        ids_a = None if ids is None else _u32(ids)
        raw_a = None if raw_ids is None else _u64(raw_ids)
        st = self.lib.or_profile_counts(
            C_.c_uint32(J), _ptr(tid), _ptr(hs), C_.c_uint64(num_samples),
            C_.c_uint64(rs.size), _ptr(rs), _ptr(rt), _ptr(ro), _ptr(rl),
            _ptr(ids_a), _ptr(raw_a), C_.c_double(rate), C_.c_uint64(seed),
            _ptr(counts), _ptr(present), _ptr(acc), C_.byref(nsel))
        if st:
            raise OracleError(st)
        out = []
        base = 0
        for j in range(J):
            H = int(hs[j])
            c = counts[base:base + H]
            total = int(acc[j])
            cap = max(1, min(H, total))
            rows = np.empty(cap, np.uint32)
            cdf = np.empty(cap, np.float64)
            icdf = np.empty(101, np.uint64)
            d = C_.c_uint64()
            self.lib.or_rank_table(_ptr(c), C_.c_uint64(H), C_.c_uint64(total),
                                   _ptr(rows), _ptr(cdf), _ptr(icdf), C_.byref(d))
            n = int(d.value)
            pres = int(present[j])
            rec = dict(table_id=int(tid[j]),
                       coverage=float(pres) / float(nsel.value),
                       avg_pooling=(float(total) / float(pres)) if pres else 0.0,
                       distinct_rows_accessed=n, total_accesses=total,
                       icdf_steps=icdf.copy(), access_cdf=cdf[:n].copy(),
                       rows_by_rank=rows[:n].copy())
            if with_counts:
                rec["counts"] = c.copy()
            out.append(rec)
            base += H
        return out

    def build_icdf(self, counts):
        c = _u64(counts)
        out = np.empty(101, np.uint64)
        st = self.lib.or_build_icdf(_ptr(c), C_.c_uint64(c.size), _ptr(out))
        if st:
            raise OracleError(st, "all access counts are zero")
        return out

    def build_remap(self, hash_size, hbm_rows, rows_by_rank, omit_unaccessed=False):
        rbr = _u32(rows_by_rank)
        ent = np.empty(max(1, hash_size), np.int32)
        slow = C_.c_uint64()
        st = self.lib.or_build_remap(C_.c_uint64(hash_size), C_.c_uint64(hbm_rows),
                                     _ptr(rbr), C_.c_uint64(rbr.size),
                                     C_.c_int(int(omit_unaccessed)), _ptr(ent),
                                     C_.byref(slow))
        if st:
            raise OracleError(st)
        return ent[:hash_size], int(slow.value)

    def simulate_counts(self, tables, rec_sample, rec_table, rec_offset,
                        rec_len, ids, table_gpu, remaps, num_gpus, sample_limit):
        J = len(tables)
        tid = _u32([t.table_id for t in tables])
        rs, rt, ro, rl, ii = (_u64(rec_sample), _u32(rec_table), _u64(rec_offset),
                              _u32(rec_len), _u32(ids))
        tg = _u32(table_gpu)
        rem = [np.ascontiguousarray(r, np.int32) for r in remaps]
        arr = (_P * J)(*[r.ctypes.data for r in rem])
        hbm = np.zeros(num_gpus, np.uint64)
        uvm = np.zeros(num_gpus, np.uint64)
        tf = np.zeros(J, np.uint64)
        tt = np.zeros(J, np.uint64)
        st = self.lib.or_simulate_counts(
            C_.c_uint32(J), _ptr(tid), C_.c_uint64(rs.size), _ptr(rs), _ptr(rt),
            _ptr(ro), _ptr(rl), _ptr(ii), _ptr(tg), arr, C_.c_uint32(num_gpus),
            C_.c_uint64(sample_limit), _ptr(hbm), _ptr(uvm), _ptr(tf), _ptr(tt))
        if st:
            raise OracleError(st)
        return hbm, uvm, tf, tt

    def init_table(self, seed, table_id, H, D, scale):
        W = np.empty((H, D), np.float32)
        self.lib.or_init_table(C_.c_uint64(seed), C_.c_uint32(table_id),
                               C_.c_uint64(H), C_.c_uint32(D), C_.c_float(scale),
                               _ptr(W))
        return W

    def emb_forward(self, B, dims, offsets, indices, weights):
        T = len(dims)
        D = _u32(dims)
        col = _u64(np.concatenate([[0], np.cumsum(dims)[:-1]]))
        stride = int(np.sum(dims))
        out = np.empty((B, stride), np.float32)
        off = _u64(offsets)
        idx = _u32(indices)
        Ws = [np.ascontiguousarray(w, np.float32) for w in weights]
        arr = (_P * T)(*[w.ctypes.data for w in Ws])
        st = self.lib.or_emb_forward(C_.c_uint32(T), C_.c_uint64(B), _ptr(D), _ptr(col),
                                     C_.c_uint64(stride), _ptr(off), _ptr(idx), arr,
                                     _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def emb_backward(self, B, dims, offsets, indices, grad_out, weights,
                     momentum, opt, lr, eps, remaps=None):
        """Updates ``weights`` / ``momentum`` (lists of numpy arrays) in place.
        ``remaps``: per table (entries int32[H], hbm_rows) of the operator's
        placement — lookups are reduced in storage-slot order; None = identity."""
        T = len(dims)
        D = _u32(dims)
        Hs = _u64([w.shape[0] for w in weights])
        col = _u64(np.concatenate([[0], np.cumsum(dims)[:-1]]))
        stride = int(np.sum(dims))
        g = np.ascontiguousarray(grad_out, np.float32)
        off = _u64(offsets)
        idx = _u32(indices)
        for w in weights:
            assert w.flags.c_contiguous and w.dtype == np.float32
        wa = (_P * T)(*[w.ctypes.data for w in weights])
        if momentum is None:
            momentum = [np.zeros(1, np.float32) for _ in weights]
        ma = (_P * T)(*[m.ctypes.data for m in momentum])
        ra, hb = None, None
        if remaps is not None:
            ents = [np.ascontiguousarray(r[0], np.int32) for r in remaps]
            ra = (_P * T)(*[e.ctypes.data for e in ents])
            hb = _u64([r[1] for r in remaps])
        st = self.lib.or_emb_backward(C_.c_uint32(T), C_.c_uint64(B), _ptr(D), _ptr(Hs),
                                      _ptr(col), C_.c_uint64(stride), _ptr(off), _ptr(idx),
                                      _ptr(g), C_.c_int(opt), C_.c_float(lr),
                                      C_.c_float(eps), wa, ma, ra, _ptr(hb))
        if st:
            raise OracleError(st)


# --------------------------------------------------------------------------
# the unmodified reference library
# --------------------------------------------------------------------------
@dataclass
class RefTrace:
    """Python view of a reference ``shardplan::Trace`` (inc/workload.hpp:41-58)."""
    tables: list
    num_samples: int
    rec_sample: np.ndarray
    rec_table: np.ndarray
    rec_offset: np.ndarray
    rec_len: np.ndarray
    ids: np.ndarray
    raw_ids: np.ndarray | None = None
    distinct_raw: np.ndarray | None = None
    handle: object = field(default=None, repr=False)


@dataclass
class _Spec:
    table_id: int
    cardinality: int
    hash_size: int
    dim: int
    elem_bytes: int


class _RefLib:
    def __init__(self, path=None):
        path = path or os.path.join(_HERE, "_ref", "libshardplan_ref.so")
        if not os.path.exists(path):
            raise OSError(f"reference oracle not built: {path}")
        L = self.lib = C_.CDLL(path)
        L.refc_last_error.restype = C_.c_char_p
        L.refc_hash_value.argtypes = [C_.c_uint64, C_.c_uint64, _P]
        L.refc_trace_free.argtypes = [_P]
        L.refc_stats_free.argtypes = [_P]
        L.refc_plan_free.argtypes = [_P]
        L.refc_trace_sizes.argtypes = [_P, _P, _P, _P]
        L.refc_stats_count.argtypes = [_P]
        L.refc_plan_size.argtypes = [_P, _P, _P, _P]

    def _chk(self, st):
        if st:
            raise OracleError(st, self.lib.refc_last_error().decode())

    def hash_value(self, raw, H):
        out = C_.c_uint32()
        self._chk(self.lib.refc_hash_value(raw, H, C_.byref(out)))
        return int(out.value)

    @staticmethod
    def _spec_arrays(specs):
        return (_u32([s.table_id for s in specs]), _u64([s.cardinality for s in specs]),
                _u64([s.hash_size for s in specs]), _u32([s.dim for s in specs]),
                _u32([s.elem_bytes for s in specs]))

    def _materialise(self, h, specs, num_samples, raw=False, gen=False):
        R, N, NR = C_.c_uint64(), C_.c_uint64(), C_.c_uint64()
        self.lib.refc_trace_sizes(h, C_.byref(R), C_.byref(N), C_.byref(NR))
        R, N, NR = int(R.value), int(N.value), int(NR.value)
        rs, rt = np.empty(R, np.uint64), np.empty(R, np.uint32)
        ro, rl = np.empty(R, np.uint64), np.empty(R, np.uint32)
        ids = np.empty(N, np.uint32)
        raws = np.empty(NR, np.uint64) if raw else None
        dr = np.zeros(len(specs), np.uint64) if gen else None
        self.lib.refc_trace_copy(h, _ptr(rs), _ptr(rt), _ptr(ro), _ptr(rl),
                                 _ptr(ids), _ptr(raws), _ptr(dr))
        return RefTrace(list(specs), num_samples, rs, rt, ro, rl, ids, raws, dr, h)

    def generate_trace(self, workload, num_samples, seed, gen_stats=False, raw=False):
        """workload: list of (TableSpec-like, (zipf, mean_pool, coverage, law))."""
        specs = [w[0] for w in workload]
        tid, card, hs, dim, eb = self._spec_arrays(specs)
        z = np.array([w[1][0] for w in workload], np.float64)
        mp = np.array([w[1][1] for w in workload], np.float64)
        cv = np.array([w[1][2] for w in workload], np.float64)
        law = np.array([w[1][3] for w in workload], np.int32)
        h = _P()
        fn = self.lib.refc_generate_raw_trace if raw else self.lib.refc_generate_trace
        args = [C_.c_uint32(len(specs)), _ptr(tid), _ptr(card), _ptr(hs), _ptr(dim),
                _ptr(eb), _ptr(z), _ptr(mp), _ptr(cv), _ptr(law),
                C_.c_uint64(num_samples), C_.c_uint64(seed)]
        if not raw:
            args.append(C_.c_int(int(gen_stats)))
        self._chk(fn(*args, C_.byref(h)))
        return self._materialise(h, specs, num_samples, raw=raw, gen=gen_stats)

    def trace(self, tables, num_samples, rec_sample, rec_table, rec_offset, rec_len, ids):
        tid, card, hs, dim, eb = self._spec_arrays(tables)
        rs, rt, ro, rl, ii = (_u64(rec_sample), _u32(rec_table), _u64(rec_offset),
                              _u32(rec_len), _u32(ids))
        h = _P()
        self._chk(self.lib.refc_trace_from_arrays(
            C_.c_uint32(len(tables)), _ptr(tid), _ptr(card), _ptr(hs), _ptr(dim), _ptr(eb),
            C_.c_uint64(num_samples), C_.c_uint64(rs.size), _ptr(rs), _ptr(rt), _ptr(ro),
            _ptr(rl), C_.c_uint64(ii.size), _ptr(ii), C_.byref(h)))
        return RefTrace(list(tables), num_samples, rs, rt, ro, rl, ii, None, None, h)

    def read_trace(self, path):
        """core/src/trace_io.cpp:75-158 (unmodified reference)."""
        h = _P()
        self._chk(self.lib.refc_read_trace(str(path).encode(), C_.byref(h)))
        J, ns = C_.c_uint32(), C_.c_uint64()
        self.lib.refc_trace_meta(h, C_.byref(J), C_.byref(ns), None, None, None, None, None)
        J = int(J.value)
        tid, card, hs = np.empty(J, np.uint32), np.empty(J, np.uint64), np.empty(J, np.uint64)
        dim, eb = np.empty(J, np.uint32), np.empty(J, np.uint32)
        if J:
            self.lib.refc_trace_meta(h, C_.byref(C_.c_uint32()), C_.byref(ns), _ptr(tid), _ptr(card),
                                     _ptr(hs), _ptr(dim), _ptr(eb))
        from types import SimpleNamespace

        specs = [SimpleNamespace(table_id=int(tid[j]), cardinality=int(card[j]), hash_size=int(hs[j]),
                                 dim=int(dim[j]), elem_bytes=int(eb[j])) for j in range(J)]
        return self._materialise(h, specs, int(ns.value))

    def write_trace(self, tr, path, comments=()):
        """core/src/trace_io.cpp:48-72 (unmodified reference); tr: a RefTrace."""
        cs = [str(c).encode() for c in comments]
        arr = (C_.c_char_p * max(1, len(cs)))(*cs)
        self._chk(self.lib.refc_write_trace(tr.handle, str(path).encode(), arr, C_.c_uint32(len(cs))))

    def free_trace(self, tr):
        if tr.handle is not None:
            self.lib.refc_trace_free(tr.handle)
            tr.handle = None

    def _stats_list(self, h):
        n = self.lib.refc_stats_count(h)
        out = []
        for j in range(n):
            tid, d, t = C_.c_uint32(), C_.c_uint64(), C_.c_uint64()
            cov, pool = C_.c_double(), C_.c_double()
            self.lib.refc_stats_scalars(h, C_.c_uint32(j), C_.byref(tid), C_.byref(cov),
                                        C_.byref(pool), C_.byref(d), C_.byref(t))
            D = int(d.value)
            icdf = np.empty(101, np.uint64)
            cdf = np.empty(D, np.float64)
            rbr = np.empty(D, np.uint32)
            self.lib.refc_stats_arrays(h, C_.c_uint32(j), _ptr(icdf), _ptr(cdf), _ptr(rbr))
            out.append(dict(table_id=int(tid.value), coverage=cov.value,
                            avg_pooling=pool.value, distinct_rows_accessed=D,
                            total_accesses=int(t.value), icdf_steps=icdf,
                            access_cdf=cdf, rows_by_rank=rbr))
        return out

    def profile(self, tr, rate, seed, keep_handle=False):
        h = _P()
        self._chk(self.lib.refc_profile(tr.handle, C_.c_double(rate),
                                        C_.c_uint64(seed), C_.byref(h)))
        stats = self._stats_list(h)
        if keep_handle:
            return stats, h
        self.lib.refc_stats_free(h)
        return stats

    def time_profile(self, tr, rate, seed):
        secs = C_.c_double()
        self._chk(self.lib.refc_time_profile(tr.handle, C_.c_double(rate),
                                             C_.c_uint64(seed), C_.byref(secs)))
        return secs.value

    def stats_handle(self, stats):
        h = _P()
        self.lib.refc_stats_new(C_.c_uint32(len(stats)), C_.byref(h))
        for j, s in enumerate(stats):
            icdf = _u64(s["icdf_steps"])
            cdf = np.ascontiguousarray(s["access_cdf"], np.float64)
            rbr = _u32(s["rows_by_rank"])
            self.lib.refc_stats_set(h, C_.c_uint32(j), C_.c_uint32(s["table_id"]),
                                    C_.c_double(s["coverage"]), C_.c_double(s["avg_pooling"]),
                                    C_.c_uint64(s["distinct_rows_accessed"]),
                                    C_.c_uint64(s["total_accesses"]), _ptr(icdf),
                                    _ptr(cdf), _ptr(rbr))
        return h

    def free_stats(self, h):
        self.lib.refc_stats_free(h)

    def build_icdf(self, counts):
        c = _u64(counts)
        out = np.empty(101, np.uint64)
        self._chk(self.lib.refc_build_icdf(_ptr(c), C_.c_uint64(c.size), _ptr(out)))
        return out

    def hash_utilization(self, distinct_rows, hash_size, distinct_raw):
        s, c = C_.c_double(), C_.c_double()
        self._chk(self.lib.refc_hash_utilization(C_.c_uint64(distinct_rows),
                                                 C_.c_uint64(hash_size),
                                                 C_.c_uint64(distinct_raw),
                                                 C_.byref(s), C_.byref(c)))
        return s.value, c.value

    def build_remap(self, stats_h, j, spec, hbm_rows, omit_unaccessed=False):
        ent = np.empty(max(1, spec.hash_size), np.int32)
        slow = C_.c_uint64()
        self._chk(self.lib.refc_build_remap(
            stats_h, C_.c_uint32(j), C_.c_uint32(spec.table_id), C_.c_uint64(spec.hash_size),
            C_.c_uint32(spec.dim), C_.c_uint32(spec.elem_bytes), C_.c_uint64(hbm_rows),
            C_.c_int(int(omit_unaccessed)), _ptr(ent), C_.byref(slow)))
        return ent[:spec.hash_size], int(slow.value)

    def write_remap(self, path, table_id, hash_size, hbm_rows, entries):
        e = np.ascontiguousarray(entries, np.int32)
        self._chk(self.lib.refc_write_remap(str(path).encode(), C_.c_uint32(table_id),
                                            C_.c_uint64(hash_size), C_.c_uint64(hbm_rows),
                                            _ptr(e if e.size else np.zeros(1, np.int32))))

    def read_remap(self, path, capacity=1 << 26):
        tid, H, hbm, slow = C_.c_uint32(), C_.c_uint64(), C_.c_uint64(), C_.c_uint64()
        ent = np.empty(max(1, capacity), np.int32)
        self._chk(self.lib.refc_read_remap(str(path).encode(), C_.byref(tid), C_.byref(H),
                                           C_.byref(hbm), _ptr(ent), C_.c_uint64(capacity),
                                           C_.byref(slow)))
        return dict(table_id=int(tid.value), hash_size=int(H.value), hbm_rows=int(hbm.value),
                    entries=ent[:int(H.value)].copy(), slow_rows_allocated=int(slow.value))

    def plan(self, tr, stats_h, kind, system, cost_kind=0, step_count=100,
             time_limit=float("inf")):
        """kind: 'milp' | 'greedy' | 'ldm'; cost_kind 0 size, 1 lookup, 2 size-lookup."""
        k = {"milp": 0, "greedy": 1, "ldm": 2}[kind]
        h = _P()
        self._chk(self.lib.refc_plan(
            tr.handle, stats_h, C_.c_int(k), C_.c_int(cost_kind),
            C_.c_uint32(system.num_gpus), C_.c_uint64(system.batch_size),
            C_.c_uint64(system.cap_hbm_bytes), C_.c_uint64(system.cap_dram_bytes),
            C_.c_double(system.bw_hbm), C_.c_double(system.bw_uvm),
            C_.c_uint32(step_count), C_.c_double(time_limit), C_.byref(h)))
        n, sc, obj = C_.c_uint32(), C_.c_uint32(), C_.c_double()
        self.lib.refc_plan_size(h, C_.byref(n), C_.byref(sc), C_.byref(obj))
        n = int(n.value)
        tid, gpu, step = np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.uint32)
        hbm, pct, mem = np.empty(n, np.uint64), np.empty(n, np.float64), np.empty(n, np.uint64)
        self.lib.refc_plan_entries(h, _ptr(tid), _ptr(gpu), _ptr(step), _ptr(hbm),
                                   _ptr(pct), _ptr(mem))
        self.lib.refc_plan_free(h)
        return dict(step_count=int(sc.value), objective=obj.value, table_id=tid, gpu=gpu,
                    step=step, hbm_rows=hbm, pct=pct, mem_bytes=mem)

    def simulate(self, tr, plan_entries, remaps, system, batch_size, timed=False):
        """plan_entries: (table_id[], gpu[], hbm_rows[]); remaps: list of
        (table_id, hash_size, hbm_rows, entries int32[])."""
        et, eg, eh = (_u32(plan_entries[0]), _u32(plan_entries[1]), _u64(plan_entries[2]))
        rt = _u32([r[0] for r in remaps])
        rh = _u64([r[1] for r in remaps])
        rb = _u64([r[2] for r in remaps])
        ents = [np.ascontiguousarray(r[3], np.int32) for r in remaps]
        arr = (_P * len(ents))(*[e.ctypes.data for e in ents])
        M = system.num_gpus
        gh, gu, gc = np.empty(M), np.empty(M), np.empty(M)
        batches, total = C_.c_uint64(), C_.c_uint64()
        agg = np.empty(5)
        tff = np.empty(len(tr.tables))
        secs = C_.c_double()
        self._chk(self.lib.refc_simulate(
            tr.handle, C_.c_uint32(et.size), _ptr(et), _ptr(eg), _ptr(eh),
            C_.c_uint32(len(ents)), _ptr(rt), _ptr(rh), _ptr(rb), arr,
            C_.c_uint32(M), C_.c_uint64(system.batch_size),
            C_.c_uint64(system.cap_hbm_bytes), C_.c_uint64(system.cap_dram_bytes),
            C_.c_double(system.bw_hbm), C_.c_double(system.bw_uvm),
            C_.c_uint64(batch_size), _ptr(gh), _ptr(gu), _ptr(gc), C_.byref(batches),
            C_.byref(total), _ptr(agg), _ptr(tff), C_.byref(secs)))
        rep = dict(hbm_accesses=gh, uvm_accesses=gu, est_iter_cost=gc,
                   batches=int(batches.value), total_accesses=int(total.value),
                   min_cost=agg[0], max_cost=agg[1], mean_cost=agg[2],
                   stddev_cost=agg[3], uvm_access_fraction=agg[4],
                   table_fast_fraction=tff)
        if timed:
            rep["seconds"] = secs.value
        return rep


def trace_to_csr(tr, table_ids, B, sample_base=0):
    """A reference Trace (records sorted by (sample, table), inc/workload.hpp:41-58)
    regrouped as the operator's table-major CSR batch: offsets u64[T*B+1]
    (bag (t, b) = samples sample_base + b), indices u32 in per-table sample order."""
    T = len(table_ids)
    tid = np.asarray(table_ids, np.uint32)
    tix = np.searchsorted(tid, tr.rec_table)
    s = tr.rec_sample.astype(np.int64) - sample_base
    keep = (s >= 0) & (s < B)
    tix, s = tix[keep], s[keep]
    st, ln = tr.rec_offset[keep].astype(np.int64), tr.rec_len[keep].astype(np.int64)
    lens = np.zeros((T, B), np.uint64)
    lens[tix, s] = ln
    offsets = np.concatenate([[0], np.cumsum(lens.ravel())]).astype(np.uint64)
    order = np.lexsort((s, tix))
    st, ln = st[order], ln[order]
    n = int(ln.sum())
    pos = np.repeat(st - np.concatenate([[0], np.cumsum(ln)[:-1]]), ln) + np.arange(n)
    return offsets, np.ascontiguousarray(tr.ids[pos], np.uint32)


def emb_step_cpu(B, dims, hash_sizes, offsets, indices, weights, momentum, opt, lr, eps,
                 threads):
    """One oracle fwd + (grad = pooled) + bwd over all tables, tables spread over
    `threads` host threads (ctypes releases the GIL).  Used only by bench.py's
    CPU baseline / reference arm.  Returns the pooled output."""
    from concurrent.futures import ThreadPoolExecutor

    c = C()
    T = len(dims)
    offsets = np.ascontiguousarray(offsets, np.uint64)
    indices = np.ascontiguousarray(indices, np.uint32)
    cols = np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int64)
    stride = int(np.sum(dims))
    pooled = np.zeros((B, stride), np.float32)

    def one(t):
        o = offsets[t * B:(t + 1) * B + 1]
        lo, hi = int(o[0]), int(o[-1])
        ot = np.ascontiguousarray(o - o[0])
        it = np.ascontiguousarray(indices[lo:hi])
        y = c.emb_forward(B, [dims[t]], ot, it, [weights[t]])
        pooled[:, cols[t]:cols[t] + dims[t]] = y
        c.emb_backward(B, [dims[t]], ot, it, y, [weights[t]],
                       None if momentum is None else [momentum[t]], opt, lr, eps)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, range(T)))
    return pooled


_c = None
_r = None


def C():
    """The plain-C restatement (always available once ``make -C oracle`` ran)."""
    global _c
    if _c is None:
        _c = _COracle()
    return _c


def Ref():
    """The compiled reference library, or raises OSError if it was never built."""
    global _r
    if _r is None:
        _r = _RefLib()
    return _r


def ref_available():
    return os.path.exists(os.path.join(_HERE, "_ref", "libshardplan_ref.so"))


Spec = _Spec
