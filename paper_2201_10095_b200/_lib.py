"""ctypes binding of ``libshardplan_gpu.so`` (the C-ABI in include/shardplan_gpu.h).

Loading fails loudly when the library is missing: there is no CPU fallback
for any hot path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RS_LIB_PATH") or os.path.join(_HERE, "libshardplan_gpu.so")

RS_OK = 0
RS_ERR_INVALID_ARGUMENT = -1
RS_ERR_PARSE = -2
RS_ERR_INFEASIBLE = -3
RS_ERR_IO = -4
RS_ERR_OUT_OF_RANGE = -5
RS_ERR_CUDA = -8
RS_ERR_INTERNAL = -9
RS_MEM_HOST = 0
RS_MEM_DEVICE = 1
RS_OPT_SGD = 0
RS_OPT_ROWWISE_ADAGRAD = 1
RS_EX_PEER = 0
RS_EX_NCCL = 1
RS_EX_BLOB_BYTES = 128

P = C.c_void_p
u32, u64, f64, f32, i32 = C.c_uint32, C.c_uint64, C.c_double, C.c_float, C.c_int


class rs_table_spec(C.Structure):
    _fields_ = [("table_id", u32), ("cardinality", u64), ("hash_size", u64),
                ("dim", u32), ("elem_bytes", u32)]


class rs_trace(C.Structure):
    _fields_ = [("num_tables", u32), ("tables", C.POINTER(rs_table_spec)),
                ("num_samples", u64), ("num_records", u64), ("rec_sample", P),
                ("rec_table", P), ("rec_offset", P), ("rec_len", P), ("num_ids", u64),
                ("ids", P), ("raw_ids", P), ("location", i32)]


class rs_feature_stats(C.Structure):
    _fields_ = [("table_id", u32), ("coverage", f64), ("avg_pooling", f64),
                ("distinct_rows_accessed", u64), ("total_accesses", u64),
                ("icdf_steps", C.POINTER(u64)), ("access_cdf", C.POINTER(f64)),
                ("rows_by_rank", C.POINTER(u32)), ("d_rows_by_rank", P)]


class rs_plan_entry(C.Structure):
    _fields_ = [("table_id", u32), ("gpu", u32), ("step", u32), ("hbm_rows", u64),
                ("pct", f64), ("mem_bytes", u64)]


class rs_system_spec(C.Structure):
    _fields_ = [("num_gpus", u32), ("batch_size", u64), ("cap_hbm_bytes", u64),
                ("cap_dram_bytes", u64), ("bw_hbm", f64), ("bw_uvm", f64)]


class rs_remap_view(C.Structure):
    _fields_ = [("table_id", u32), ("hash_size", u64), ("hbm_rows", u64), ("entries", P),
                ("location", i32)]


class rs_sim_report(C.Structure):
    _fields_ = [("gpu_hbm_accesses", C.POINTER(f64)), ("gpu_uvm_accesses", C.POINTER(f64)),
                ("gpu_est_iter_cost", C.POINTER(f64)), ("batches", u64),
                ("total_accesses", u64), ("min_cost", f64), ("max_cost", f64),
                ("mean_cost", f64), ("stddev_cost", f64), ("uvm_access_fraction", f64),
                ("table_fast_fraction", C.POINTER(f64))]


class rs_emb_table(C.Structure):
    _fields_ = [("table_id", u32), ("hash_size", u64), ("dim", u32), ("remap", P),
                ("remap_location", i32), ("hbm_rows", u64), ("slow_rows", u64),
                ("elem_bytes", u32), ("allow_unbacked", i32)]


class rs_plan_table(C.Structure):
    _fields_ = [("spec", rs_table_spec), ("coverage", f64), ("avg_pooling", f64),
                ("icdf_steps", P)]


class rs_plan_summary(C.Structure):
    _fields_ = [("objective", f64), ("lower_bound", f64), ("proved_optimal", i32)]


class rs_gen_table(C.Structure):
    _fields_ = [("table_id", u32), ("cardinality", u64), ("hash_size", u64),
                ("zipf_exponent", f64), ("mean_pooling", f64), ("coverage", f64),
                ("pooling_law", i32)]


_SIGS = {
    "rs_abi_version": ([], i32),
    "rs_launch_counter": ([], u64),
    "rs_last_error": ([], C.c_char_p),
    "rs_context_create": ([i32, P, i32, P], i32),
    "rs_context_destroy": ([P], i32),
    "rs_context_synchronize": ([P], i32),
    "rs_hash_value": ([u64, u64, P], i32),
    "rs_hash_ids": ([P, P, u64, u64, P, i32], i32),
    "rs_profile_run": ([P, P, f64, u64, P], i32),
    "rs_profile_num_tables": ([P, P], i32),
    "rs_profile_get": ([P, u32, P], i32),
    "rs_profile_selected": ([P, P], i32),
    "rs_profile_destroy": ([P], i32),
    "rs_build_icdf": ([P, P, u64, i32, P], i32),
    "rs_hash_utilization": ([u64, u64, u64, P, P], i32),
    "rs_count_distinct_raw": ([P, P, P], i32),
    "rs_build_remap": ([P, u32, u64, u64, P, u64, i32, i32, P, i32, P], i32),
    "rs_simulate": ([P, P, u32, P, u32, P, P, u64, P], i32),
    "rs_emb_create": ([P, u32, P, u64, u64, i32, f32, P], i32),
    "rs_emb_destroy": ([P], i32),
    "rs_emb_init_weights": ([P, u64, f32], i32),
    "rs_emb_forward": ([P, u64, P, P, P, P], i32),
    "rs_emb_backward": ([P, u64, P, P, P, f32], i32),
    "rs_emb_read_rows": ([P, u32, P, u64, P, P], i32),
    "rs_emb_enable_uvm_cache": ([P, u32], i32),
    "rs_emb_prefetch": ([P, u64, P, P], i32),
    "rs_emb_flush": ([P], i32),
    "rs_emb_memory": ([P, P, P], i32),
    "rs_emb_unbacked": ([P, P, P, i32], i32),
    "rs_emb_kernel_times": ([P, P, P, P, P, i32], i32),
    "rs_remap_write": ([P, C.c_char_p, u32, u64, u64, P, i32], i32),
    "rs_trace_read": ([P, C.c_char_p, u64, P], i32),
    "rs_trace_file_view": ([P, P], i32),
    "rs_trace_file_export": ([P, P, P, P, P, P, P, i32], i32),
    "rs_trace_file_destroy": ([P], i32),
    "rs_trace_write": ([P, P, C.c_char_p, P, u32], i32),
    "rs_remap_read_header": ([C.c_char_p, P, P, P], i32),
    "rs_remap_read": ([P, C.c_char_p, P, i32, u64, P], i32),
    "rs_radix_sort_pairs": ([P, P, P, u64, i32], i32),
    "rs_gen_batch": ([P, u32, P, u64, u64, u64, P, P, u64, P], i32),
    "rs_kjt_to_records": ([P, u32, P, u64, u64, P, P, P, P, P, P], i32),
    "rs_plan_last_error": ([], C.c_char_p),
    "rs_table_fixed_cost": ([P, P, i32, P], i32),
    "rs_plan_greedy": ([u32, P, P, P, P, P, P], i32),
    "rs_plan_ldm": ([u32, P, P, P, P, P, P], i32),
    "rs_plan_solve": ([u32, P, P, u32, i32, i32, f64, u32, P, P, P], i32),
    "rs_exchange_create": ([P, i32, u32, u32, u64, u32, P, P, P], i32),
    "rs_exchange_blob": ([P, P], i32),
    "rs_exchange_connect": ([P, P], i32),
    "rs_exchange_info": ([P, P, P, P, P], i32),
    "rs_exchange_destroy": ([P], i32),
    "rs_emb_forward_to_owners": ([P, P, P, P, P, P], i32),
    "rs_emb_backward_from_owners": ([P, P, P, P, P, f32], i32),
    "rs_emb_alltoall_fwd": ([P, P, P], i32),
    "rs_emb_alltoall_bwd": ([P, P, P], i32),
}

# every symbol include/shardplan_gpu.h declares (checked by the CPU test suite)
EXPORTS = tuple(_SIGS)

_lib = None


def lib():
    """The loaded product library (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2201_10095_b200/csrc` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(status, planner=False):
    """Raise the reference's exception type for a negative status."""
    if status == RS_OK:
        return
    from .types import error_for_status
    msg = lib().rs_plan_last_error() if planner else lib().rs_last_error()
    raise error_for_status(status, msg.decode() if msg else "")
