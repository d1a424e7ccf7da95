/* shardplan_gpu — C-ABI of the B200-native RecShard hot paths.
 *
 * The drop-in boundary: plain pointers, sizes and opaque handles, no torch or
 * C++ types.  Every entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/core/).  The C++ shim
 * include/shardplan_gpu.hpp rebuilds the reference's `shardplan::` value API
 * (profile / build_icdf / hash_utilization / hash_value / build_remap /
 * translate / simulate) on top of it and rethrows the reference's exception
 * types.
 *
 * Conventions
 *  - Return value: RS_OK (0) or a negative RS_ERR_* status; the message of the
 *    last failure on this thread is rs_last_error().
 *  - `location` arguments say where a buffer lives: RS_MEM_HOST (pageable or
 *    pinned host memory; staged over PCIe inside the call) or RS_MEM_DEVICE
 *    (device memory of the context's GPU).
 *  - Calls are ordered on the context's stream.  Calls that return host
 *    results synchronise that stream before returning; rs_emb_* calls on
 *    device buffers are asynchronous.
 *  - One context per stream/thread; concurrent calls must use distinct
 *    contexts (the reference functions are pure and re-entrant).
 */
#ifndef SHARDPLAN_GPU_H
#define SHARDPLAN_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 1

/* Status codes — mirror include/shardplan/error.hpp:38-72. */
#define RS_OK 0
#define RS_ERR_INVALID_ARGUMENT (-1) /* shardplan::InvalidArgument          */
#define RS_ERR_PARSE (-2)            /* shardplan::ParseError               */
#define RS_ERR_INFEASIBLE (-3)       /* shardplan::InfeasibleError          */
#define RS_ERR_IO (-4)               /* shardplan::IoError                  */
#define RS_ERR_OUT_OF_RANGE (-5)     /* std::out_of_range (profiler.cpp:103) */
#define RS_ERR_CUDA (-8)             /* CUDA runtime failure                */
#define RS_ERR_INTERNAL (-9)

#define RS_MEM_HOST 0
#define RS_MEM_DEVICE 1

#define RS_OPT_SGD 0               /* row-wise SGD                          */
#define RS_OPT_ROWWISE_ADAGRAD 1   /* FBGEMM exact row-wise Adagrad         */

int rs_abi_version(void);
const char* rs_last_error(void);
/* Kernel launches issued by this library so far (process-wide diagnostic). */
uint64_t rs_launch_counter(void);

/* ------------------------------------------------------------- context */
typedef struct rs_context rs_context;
/* Runs on `stream` (a cudaStream_t; NULL = the legacy default stream), or on
 * a private non-blocking stream when flags has RS_CTX_PRIVATE_STREAM. */
#define RS_CTX_PRIVATE_STREAM 1
int rs_context_create(int device, void* stream, int flags, rs_context** out);
int rs_context_destroy(rs_context* ctx);
int rs_context_synchronize(rs_context* ctx);

/* ------------------------------------------------------------- types  */
/* include/shardplan/types.hpp:26-34 (TableSpec) */
typedef struct rs_table_spec {
  uint32_t table_id;
  uint64_t cardinality;
  uint64_t hash_size;
  uint32_t dim;
  uint32_t elem_bytes;
} rs_table_spec;

/* include/shardplan/workload.hpp:41-58 (Trace) in structure-of-arrays form.
 * Exactly one of `ids` (hashed rows) and `raw_ids` (pre-hash values, hashed
 * on the GPU with hash_value's mix64 % hash_size) is non-NULL. */
typedef struct rs_trace {
  uint32_t num_tables;
  const rs_table_spec* tables; /* host */
  uint64_t num_samples;
  uint64_t num_records;
  const uint64_t* rec_sample;
  const uint32_t* rec_table; /* table_id, not index */
  const uint64_t* rec_offset;
  const uint32_t* rec_len;
  uint64_t num_ids;
  const uint32_t* ids;
  const uint64_t* raw_ids;
  int location; /* of the record and id arrays */
} rs_trace;

/* ------------------------------------------------------------- hashing */
/* include/shardplan/workload.hpp:28-31  hash_value(raw, hash_size) */
int rs_hash_value(uint64_t raw_id, uint64_t hash_size, uint32_t* out);
/* Batched hash_value on the GPU (K0).  raw/out: `location` buffers. */
int rs_hash_ids(rs_context* ctx, const uint64_t* raw, uint64_t n,
                uint64_t hash_size, uint32_t* out, int location);

/* ------------------------------------------------------------- profiler */
typedef struct rs_profile rs_profile;

/* core/src/profiler.cpp:60-161  profile(trace, sample_rate, seed).
 * K1 (select + hash + histogram) and K2 (rank, CDF, ICDF) run on the GPU.
 * Errors as the reference: empty trace / rate outside (0,1] / zero samples
 * selected -> RS_ERR_INVALID_ARGUMENT; a selected record of an unknown
 * table -> RS_ERR_OUT_OF_RANGE. */
int rs_profile_run(rs_context* ctx, const rs_trace* trace, double sample_rate,
                   uint64_t seed, rs_profile** out);

/* include/shardplan/profiler.hpp:31-45 (FeatureStats) view. Pointers stay
 * valid until rs_profile_destroy. */
typedef struct rs_feature_stats {
  uint32_t table_id;
  double coverage;
  double avg_pooling;
  uint64_t distinct_rows_accessed;
  uint64_t total_accesses;
  const uint64_t* icdf_steps;      /* 101 entries, host */
  const double* access_cdf;        /* distinct entries, host */
  const uint32_t* rows_by_rank;    /* distinct entries, host */
  const uint32_t* d_rows_by_rank;  /* same, device (feeds rs_build_remap) */
} rs_feature_stats;

int rs_profile_num_tables(const rs_profile* p, uint32_t* out);
int rs_profile_get(const rs_profile* p, uint32_t j, rs_feature_stats* out);
/* Number of selected samples (the coverage denominator, profiler.cpp:68-76). */
int rs_profile_selected(const rs_profile* p, uint64_t* out);
int rs_profile_destroy(rs_profile* p);

/* core/src/profiler.cpp:49-58  build_icdf(counts) on the GPU (sort + scan).
 * counts: `location` buffer of n u64; out: host u64[101]. */
int rs_build_icdf(rs_context* ctx, const uint64_t* counts, uint64_t n,
                  int location, uint64_t* out101);

/* GenStats.distinct_raw_ids (include/shardplan/workload.hpp:62-64,
 * core/src/workload.cpp:195-223) for a raw trace: distinct raw values per
 * table over every record (GPU hash sets).  out: host u64[num_tables]. */
int rs_count_distinct_raw(rs_context* ctx, const rs_trace* trace, uint64_t* out);

/* core/src/profiler.cpp:163-174  hash_utilization(stats, spec, distinct_raw) */
int rs_hash_utilization(uint64_t distinct_rows_accessed, uint64_t hash_size,
                        uint64_t distinct_raw_ids_seen, double* sparsity,
                        double* collisions);

/* ------------------------------------------------------------- remap   */
/* core/src/remap.cpp:40-105  build_remap(entry, stats, spec, opts) (K3).
 * rows_by_rank: `rows_location` buffer of `distinct` u32 (e.g. the device
 * view of rs_feature_stats); entries: `out_location` buffer of hash_size
 * int32 (sign-bit tier encoding, include/shardplan/remap.hpp:27-29). */
int rs_build_remap(rs_context* ctx, uint32_t table_id, uint64_t hash_size,
                   uint64_t hbm_rows, const uint32_t* rows_by_rank,
                   uint64_t distinct, int rows_location, int omit_unaccessed,
                   int32_t* entries, int out_location,
                   uint64_t* slow_rows_allocated);

/* ------------------------------------------------------------- simulate */
/* include/shardplan/plan.hpp:27-34 (PlanEntry) */
typedef struct rs_plan_entry {
  uint32_t table_id;
  uint32_t gpu;
  uint32_t step;
  uint64_t hbm_rows;
  double pct;
  uint64_t mem_bytes;
} rs_plan_entry;

/* include/shardplan/types.hpp:82-89 (SystemSpec) */
typedef struct rs_system_spec {
  uint32_t num_gpus;
  uint64_t batch_size;
  uint64_t cap_hbm_bytes;
  uint64_t cap_dram_bytes;
  double bw_hbm;
  double bw_uvm;
} rs_system_spec;

/* include/shardplan/remap.hpp:27-39 (RemapTable) */
/* SPRM remap files (include/shardplan/remap.hpp:60-63, core/src/remap.cpp:118-176),
 * byte-compatible with the reference's write_remap / read_remap.  entries /
 * out live at `location` (device reads stream through pinned memory in
 * chunks, the file read overlapping the DMA).  rs_remap_read_header sizes the
 * buffer; rs_remap_read fills it and returns the reference's
 * slow_rows_allocated (count of negative entries).  Errors: IoError (open /
 * write), ParseError (short, bad magic/version, hash_size out of range,
 * truncated) — the reference's types and messages. */
int rs_remap_write(rs_context* ctx, const char* path, uint32_t table_id, uint64_t hash_size,
                   uint64_t hbm_rows, const int32_t* entries, int location);
int rs_remap_read_header(const char* path, uint32_t* table_id, uint64_t* hash_size, uint64_t* hbm_rows);
int rs_remap_read(rs_context* ctx, const char* path, int32_t* out, int location, uint64_t capacity,
                  uint64_t* slow_rows_allocated);

/* ------------------------------------------------------------- trace files */
/* core/src/trace_io.cpp:75-158  read_trace(path) — text, or gzip for ".gz"
 * paths (core/src/line_io.cpp).  Parsed on the GPU in chunks of
 * `chunk_bytes` (0 = 64 MiB); the result stays in device memory, owned by
 * the handle.  Errors as the reference, with its messages: IoError (cannot
 * open / read failed), ParseError ("line N: ..."), InvalidArgument (unknown
 * table, sample or id out of range, unsorted records, duplicate table,
 * TableSpec validation). */
typedef struct rs_trace_file rs_trace_file;
int rs_trace_read(rs_context* ctx, const char* path, uint64_t chunk_bytes, rs_trace_file** out);
/* The loaded trace as an rs_trace (tables on the host, record and id arrays on
 * the device, location RS_MEM_DEVICE) — valid until rs_trace_file_destroy;
 * pass it straight to rs_profile_run / rs_simulate. */
int rs_trace_file_view(const rs_trace_file* f, rs_trace* view);
/* Copies the record and id arrays into caller buffers (`location`), sized
 * num_records / num_ids from the view; NULL skips an array. */
int rs_trace_file_export(rs_context* ctx, const rs_trace_file* f, uint64_t* rec_sample,
                         uint32_t* rec_table, uint64_t* rec_offset, uint32_t* rec_len,
                         uint32_t* ids, int location);
int rs_trace_file_destroy(rs_trace_file* f);
/* core/src/trace_io.cpp:48-72  write_trace(trace, path, comments): the record
 * lines are formatted on the GPU, byte-identical to the reference writer
 * (gzip through zlib for ".gz").  `trace` must carry hashed ids. */
int rs_trace_write(rs_context* ctx, const rs_trace* trace, const char* path,
                   const char* const* comments, uint32_t n_comments);

typedef struct rs_remap_view {
  uint32_t table_id;
  uint64_t hash_size;
  uint64_t hbm_rows;
  const int32_t* entries;
  int location;
} rs_remap_view;

/* include/shardplan/simulator.hpp:24-39 (SimReport); caller-owned arrays:
 * gpu_* hold num_gpus entries, table_fast_fraction num_tables. */
typedef struct rs_sim_report {
  double* gpu_hbm_accesses;
  double* gpu_uvm_accesses;
  double* gpu_est_iter_cost;
  uint64_t batches;
  uint64_t total_accesses;
  double min_cost, max_cost, mean_cost, stddev_cost;
  double uvm_access_fraction;
  double* table_fast_fraction;
} rs_sim_report;

/* core/src/simulator.cpp:26-139  simulate(trace, plan, remaps, system, B).
 * The per-GPU / per-table tier counts are exact u64 from the GPU; the
 * report formulas are applied on the host exactly as the reference does. */
int rs_simulate(rs_context* ctx, const rs_trace* trace, uint32_t num_entries,
                const rs_plan_entry* entries, uint32_t num_remaps,
                const rs_remap_view* remaps, const rs_system_spec* system,
                uint64_t batch_size, rs_sim_report* out);

/* ------------------------------------------------------------- planner (host)
 * The sharder's cost model and placements (tiny host
 * work, no GPU): bit-identical plans to the reference's, faster.  Tables are
 * (TableSpec, FeatureStats) pairs aligned by index — a MilpInstance
 * (include/shardplan/plan.hpp:37-47) — and `entries` receives one
 * rs_plan_entry per table in the same order, gpu_cost num_gpus doubles.
 * Errors: RS_ERR_INVALID_ARGUMENT / RS_ERR_INFEASIBLE with the reference's
 * messages; the message is rs_plan_last_error(). */
typedef struct rs_plan_table {
  rs_table_spec spec;
  double coverage;              /* FeatureStats.coverage */
  double avg_pooling;           /* FeatureStats.avg_pooling */
  const uint64_t* icdf_steps;   /* FeatureStats.icdf_steps, 101 entries */
} rs_plan_table;

typedef struct rs_plan_summary {
  double objective;     /* ShardingPlan.objective (max_m gpu_cost) */
  double lower_bound;   /* ShardingPlan.lower_bound */
  int proved_optimal;   /* ShardingPlan.proved_optimal */
} rs_plan_summary;

#define RS_COST_SIZE 0         /* CostKind::kSize          hash_size * dim */
#define RS_COST_LOOKUP 1       /* CostKind::kLookup        avg_pool * dim */
#define RS_COST_SIZE_LOOKUP 2  /* CostKind::kSizeAndLookup avg_pool * dim * log10(hash_size) */

const char* rs_plan_last_error(void);
/* core/src/baselines.cpp:44-67  table_fixed_cost(spec, stats, kind);
 * avg_pooling may be NULL for RS_COST_SIZE (stats == nullptr). */
int rs_table_fixed_cost(const rs_table_spec* spec, const double* avg_pooling, int kind, double* out);
/* core/src/baselines.cpp:136-203  greedy_shard(costs, specs, stats, system) */
int rs_plan_greedy(uint32_t num_tables, const rs_plan_table* tables, const double* costs,
                   const rs_system_spec* system, rs_plan_entry* entries, double* gpu_cost,
                   rs_plan_summary* summary);
/* core/src/baselines.cpp:205-292  ldm_shard(costs, specs, stats, system) */
int rs_plan_ldm(uint32_t num_tables, const rs_plan_table* tables, const double* costs,
                const rs_system_spec* system, rs_plan_entry* entries, double* gpu_cost,
                rs_plan_summary* summary);
/* core/src/milp_solve.cpp:633-709  solve(build_instance(stats, specs, system,
 * ablation, step_count), time_limit_seconds) — INFINITY for the default
 * budget.  `threads` (0 = all cores) evaluate the local search's candidate
 * moves; the plan does not depend on it. */
int rs_plan_solve(uint32_t num_tables, const rs_plan_table* tables, const rs_system_spec* system,
                  uint32_t step_count, int use_pooling, int use_coverage, double time_limit_seconds,
                  uint32_t threads, rs_plan_entry* entries, double* gpu_cost, rs_plan_summary* summary);

/* ------------------------------------------------------------- EmbeddingBag
 * The tiered operator that serves a plan (no reference implementation: the
 * paper used FBGEMM; semantics PAPER.md:275 and :605-607).
 * Each table's rows live in the fast tier (HBM) or the slow tier (pinned
 * host memory read zero-copy over PCIe) as its remap says.  Rows are fp32 or
 * fp16 (elem_bytes 2); pooling, gradients and the optimizer run in fp32.
 *
 * Batch format (table-major CSR, the reference Trace regrouped per table):
 *   offsets: u32[T*B + 1]; bag (t, b) = indices[offsets[t*B+b] .. offsets[t*B+b+1])
 *   indices: u32 ORIGINAL row ids (< hash_size); remap is applied in-kernel.
 *   pooled:  f32[B, sum_t dim_t], table t at column sum_{u<t} dim_u.      */
typedef struct rs_emb rs_emb;

typedef struct rs_emb_table {
  uint32_t table_id;
  uint64_t hash_size;
  uint32_t dim;                 /* multiple of 4, <= 1024 */
  const int32_t* remap;         /* hash_size entries, host or device */
  int remap_location;
  uint64_t hbm_rows;            /* fast-tier rows (remap >= 0) */
  uint64_t slow_rows;           /* slow-tier rows to back (remap < 0): RemapTable.slow_rows_allocated */
  uint32_t elem_bytes;          /* TableSpec.elem_bytes (inc/types.hpp:31): 4 = fp32 rows, 2 = fp16
                                   rows (fp32 arithmetic, round-to-nearest-even stores); 0 means 4 */
  int allow_unbacked;           /* 1: slow offsets >= slow_rows are rows an omit_unaccessed remap
                                   (inc/remap.hpp:43-48) left without storage — they pool as zero
                                   vectors and their gradients are dropped (rs_emb_unbacked counts
                                   them); 0: such an entry is rejected at create */
} rs_emb_table;

int rs_emb_create(rs_context* ctx, uint32_t num_tables, const rs_emb_table* tables,
                  uint64_t max_batch, uint64_t max_lookups, int optimizer, float eps,
                  rs_emb** out);
int rs_emb_destroy(rs_emb* e);
/* Deterministic init on ORIGINAL rows (oracle/oracle.h or_init_weight). */
int rs_emb_init_weights(rs_emb* e, uint64_t seed, float scale);
/* K4: sum-pooled forward.  hit_counts (device u64[2*T], may be NULL) receives
 * += per-table fast / slow lookup counts (the simulate() accounting). */
int rs_emb_forward(rs_emb* e, uint64_t batch, const uint32_t* offsets,
                   const uint32_t* indices, float* pooled, uint64_t* hit_counts);
/* K5: backward + optimizer update, deterministic (sorted-segment reduction). */
int rs_emb_backward(rs_emb* e, uint64_t batch, const uint32_t* offsets,
                    const uint32_t* indices, const float* grad_pooled, float lr);
/* HBM staging of slow-tier rows, overlapped with compute: after
 * rs_emb_enable_uvm_cache(nslots), rs_emb_prefetch(batch k+1) — called after
 * batch k's forward — lists batch k+1's slow rows that are not staged yet
 * (claim kernel on the operator's stream); a host worker gathers them from
 * the host tier and the copy engines move them into HBM slots while batch k's
 * backward runs.  The forward/backward of batch k+1 use the staged copies;
 * rows no live batch needs are evicted one step after their last use and
 * returned to the host tier the same way (DMA + host scatter).  At most two
 * prefetched batches pending; results are bit-identical to the zero-copy
 * path.  nslots should be >= 4x the unique slow rows of one batch.
 * rs_emb_flush writes every staged row back (read_rows / init_weights do so
 * implicitly). */
int rs_emb_enable_uvm_cache(rs_emb* e, uint32_t nslots);
int rs_emb_prefetch(rs_emb* e, uint64_t batch, const uint32_t* offsets, const uint32_t* indices);
int rs_emb_flush(rs_emb* e);
/* Reads rows by ORIGINAL id into host memory (parity checks). */
int rs_emb_read_rows(rs_emb* e, uint32_t t, const uint32_t* rows, uint64_t n,
                     float* out, float* momentum_out);
/* Lookups that hit unbacked rows since the last reset (per table, u64[T],
 * host), and how many remap entries of each table are unbacked (may be NULL). */
int rs_emb_unbacked(rs_emb* e, uint64_t* lookups, uint64_t* rows, int reset);
/* Bytes of HBM / pinned host memory held by the tiers. */
int rs_emb_memory(const rs_emb* e, uint64_t* hbm_bytes, uint64_t* host_bytes);
/* Kernel-only time of the forward / backward kernel sequences since the last
 * reset (CUDA events on the operator's stream around the kernels, excluding
 * slow-row staging waits), and how many calls it covers.  Synchronises. */
int rs_emb_kernel_times(rs_emb* e, double* fwd_ms, uint64_t* n_fwd, double* bwd_ms, uint64_t* n_bwd,
                        int reset);

/* ------------------------------------------------------------- K6: rank exchange
 * Table-wise model parallelism across the GPUs of one node: rank
 * r owns the tables with PlanEntry.gpu == r (both tiers)
 * and pools them for the whole global batch B; it also owns samples
 * [r*B/N, (r+1)*B/N).  An exchange moves every pooled row to its sample owner
 * ([B/N, sum of ALL dims], tables in global order) and every gradient row
 * back to its table owner ([B, sum of this rank's dims], its tables in global
 * order).  Transports: RS_EX_PEER — NVLink peer memory between the ranks'
 * processes (CUDA IPC), the forward fused into K4's stores; RS_EX_NCCL —
 * grouped ncclSend/ncclRecv (the process's libnccl.so.2, resolved at run
 * time).  Bootstrap: every rank calls rs_exchange_blob; the caller all-gathers
 * the blobs (rank-ordered, RS_EX_BLOB_BYTES each; NCCL needs only rank 0's)
 * with its own plumbing and passes them to rs_exchange_connect. */
typedef struct rs_exchange rs_exchange;
#define RS_EX_PEER 0
#define RS_EX_NCCL 1
#define RS_EX_BLOB_BYTES 128
/* dims/owner: per GLOBAL table (plan order) its dim and owner rank. */
int rs_exchange_create(rs_context* ctx, int transport, uint32_t nranks, uint32_t rank, uint64_t batch,
                       uint32_t num_tables, const uint32_t* dims, const uint32_t* owner, rs_exchange** out);
int rs_exchange_blob(rs_exchange* x, void* blob);
int rs_exchange_connect(rs_exchange* x, const void* blobs);
/* bl = B/N, d_total = sum of all dims, d_local = this rank's; owned = the
 * current step's owner block [bl, d_total] (device; valid until the next forward). */
int rs_exchange_info(const rs_exchange* x, uint64_t* bl, uint64_t* d_total, uint64_t* d_local, float** owned);
int rs_exchange_destroy(rs_exchange* x);
/* K4 + K6: this rank's operator `e` (its tables, in global order) pools the
 * batch (offsets/indices of ITS tables for all B samples) and every row lands
 * in its owner's block; *owned receives this rank's block [bl, d_total]. */
int rs_emb_forward_to_owners(rs_emb* e, rs_exchange* x, const uint32_t* offsets, const uint32_t* indices,
                             uint64_t* hit_counts, float** owned);
/* K6 + K5: the gradient of this rank's owner block (written in place into
 * *owned, or given as grad_owned [bl, d_total]) returns to the table owners on
 * a side stream while K5 plans and sorts; then K5 updates this rank's tables. */
int rs_emb_backward_from_owners(rs_emb* e, rs_exchange* x, const uint32_t* offsets, const uint32_t* indices,
                                const float* grad_owned, float lr);
/* The K6 primitives alone: pooled [B, d_local] -> owner block
 * [bl, d_total]; gradients [bl, d_total] -> [B, d_local].  Stream-ordered on
 * the exchange's context. */
int rs_emb_alltoall_fwd(rs_exchange* x, const float* pooled_local, float* pooled_owned);
int rs_emb_alltoall_bwd(rs_exchange* x, const float* grad_owned, float* grad_local);

/* ------------------------------------------------------------- primitives
 * The device-wide stable LSD radix sort behind K2 and K5 (device buffers,
 * sorted in place on bits [0, end_bit); vals may be NULL). */
int rs_radix_sort_pairs(rs_context* ctx, uint32_t* keys, uint32_t* vals, uint64_t n,
                        int end_bit);

/* ------------------------------------------------------------- synthetic workload
 * Bench/test INPUT generation — not part of the reference boundary.  Mirrors
 * core/src/workload.cpp:198-217 (per (sample, table) substream, coverage
 * Bernoulli, pooling law, bounded Zipf raw values, hash_value) on the GPU;
 * not bit-identical to the reference generator (GPU libm). */
typedef struct rs_gen_table {
  uint32_t table_id;
  uint64_t cardinality;
  uint64_t hash_size;
  double zipf_exponent;
  double mean_pooling;
  double coverage;
  int pooling_law; /* 0 constant, 1 poisson, 2 lognormal (types.hpp:57) */
} rs_gen_table;

/* Writes a table-major CSR batch (device offsets[T*B+1], indices) for samples
 * [sample_base, sample_base + B).  *total = lookups; fails without writing
 * indices if total > capacity. */
int rs_gen_batch(rs_context* ctx, uint32_t T, const rs_gen_table* tables, uint64_t B,
                 uint64_t sample_base, uint64_t seed, uint32_t* offsets, uint32_t* indices,
                 uint64_t capacity, uint64_t* total);
/* Device view of a CSR batch as reference Trace records (present bags only). */
int rs_kjt_to_records(rs_context* ctx, uint32_t T, const uint32_t* table_ids, uint64_t B,
                      uint64_t sample_base, const uint32_t* offsets, uint64_t* rec_sample,
                      uint32_t* rec_table, uint64_t* rec_offset, uint32_t* rec_len,
                      uint64_t* num_records);

#ifdef __cplusplus
}
#endif
#endif
