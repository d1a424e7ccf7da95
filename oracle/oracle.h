/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the RecShard hot paths.
 *
 * A plain-C restatement of the reference algorithms on the two hot paths,
 * used exclusively by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER.  The product library
 * (paper_2201_10095_b200/libshardplan_gpu.so) never links or calls it.
 *
 * Parity is pinned two ways (tests/test_oracle_golden.py):
 *   1. against the reference's own known-answer tests (tests/test_workload.cpp,
 *      test_profiler.cpp, test_remap.cpp, test_simulator.cpp) restated as
 *      golden fixtures in tests/golden/; and
 *   2. against the unmodified reference library compiled from
 *      /root/reference by oracle/Makefile into oracle/_ref/.
 * The EmbeddingBag forward/backward has no reference implementation (the
 * paper used FBGEMM, which is not vendored): those two functions
 * restate the paper's sum-pool definition and FBGEMM's
 * row-wise SGD / exact-row-wise-Adagrad update, with the arithmetic order
 * spelled out below — "parity unpinned" at the reference boundary for them.
 *
 * Status codes: 0 ok, -1 invalid argument (the reference's InvalidArgument),
 * -5 unknown table id (the reference lets std::out_of_range escape,
 * core/src/profiler.cpp:103).
 */
#ifndef RECSHARD_ORACLE_H
#define RECSHARD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* inc/rng.hpp:27-31 */
uint64_t or_mix64(uint64_t z);
/* inc/rng.hpp:61-64 */
uint64_t or_derive_stream(uint64_t master, uint64_t a, uint64_t b);
/* inc/workload.hpp:28-31 */
int or_hash_value(uint64_t raw, uint64_t hash_size, uint32_t* out);
int or_hash_batch(const uint64_t* raw, uint64_t n, uint64_t hash_size,
                  uint32_t* out);

/* core/src/profiler.cpp:60-112: sample selection + per-row counting.
 * counts: caller-provided, zeroed, sum(hash_size) u64 slots, table-major in
 * trace table order.  ids: hashed rows; if raw_ids != NULL the raw ids are
 * hashed first (profile_raw).  selected_out may be NULL. */
int or_profile_counts(uint32_t J, const uint32_t* table_ids,
                      const uint64_t* hash_sizes, uint64_t num_samples,
                      uint64_t R, const uint64_t* rec_sample,
                      const uint32_t* rec_table, const uint64_t* rec_offset,
                      const uint32_t* rec_len, const uint32_t* ids,
                      const uint64_t* raw_ids, double rate, uint64_t seed,
                      uint64_t* counts, uint64_t* present, uint64_t* accesses,
                      uint64_t* selected_count);

/* core/src/profiler.cpp:114-159 for one table: rank rows by (count desc,
 * row asc), cumulative CDF as double(cum)/double(total), 101-step ICDF.
 * rows_by_rank / cdf need room for min(H, total) entries. */
int or_rank_table(const uint64_t* counts, uint64_t H, uint64_t total,
                  uint32_t* rows_by_rank, double* cdf, uint64_t* icdf101,
                  uint64_t* distinct);

/* core/src/profiler.cpp:49-58 */
int or_build_icdf(const uint64_t* counts, uint64_t n, uint64_t* icdf101);

/* core/src/remap.cpp:40-105 */
int or_build_remap(uint64_t hash_size, uint64_t hbm_rows,
                   const uint32_t* rows_by_rank, uint64_t distinct,
                   int omit_unaccessed, int32_t* entries,
                   uint64_t* slow_rows_allocated);

/* core/src/simulator.cpp:72-94: exact integer tier counts.  table_gpu[j]
 * is the plan's GPU for trace table j; remaps[j] its entries. */
int or_simulate_counts(uint32_t J, const uint32_t* table_ids, uint64_t R,
                       const uint64_t* rec_sample, const uint32_t* rec_table,
                       const uint64_t* rec_offset, const uint32_t* rec_len,
                       const uint32_t* ids, const uint32_t* table_gpu,
                       const int32_t* const* remaps, uint32_t num_gpus,
                       uint64_t sample_limit, uint64_t* hbm_count,
                       uint64_t* uvm_count, uint64_t* table_fast,
                       uint64_t* table_total);

/* Deterministic weight initialisation, defined on ORIGINAL row ids so the
 * oracle can rebuild any row regardless of its tier:
 *   u = mix64(derive_stream(seed, table_id, row) + d) >> 40       (24 bits)
 *   w = ((float)u * 2^-24 - 0.5f) * scale                          */
float or_init_weight(uint64_t seed, uint32_t table_id, uint64_t row,
                     uint32_t d, float scale);
void or_init_table(uint64_t seed, uint32_t table_id, uint64_t H, uint32_t D,
                   float scale, float* W);

/* Sum-pooled EmbeddingBag forward (a NULL feature pools to 0).
 * Bags are table-major: bag (t, b) covers indices[offsets[t*B+b] ..
 * offsets[t*B+b+1]).  out is [B, sum(D)] with table t at column col_off[t].
 * Each element is accumulated in fp32 in ascending lookup order starting
 * from +0.0f (no FMA). */
int or_emb_forward(uint32_t T, uint64_t B, const uint32_t* D,
                   const uint64_t* col_off, uint64_t out_stride,
                   const uint64_t* offsets, const uint32_t* indices,
                   const float* const* W, float* out);

/* Backward + optimizer.  All lookups of the batch are ordered stably by
 * global key = (sum of earlier tables' hash sizes) + slot, where slot is the
 * row's storage slot in the operator's tiers (csrc/emb.cu keygen_kernel):
 * remap entry e >= 0 -> e, e < 0 -> hbm_rows[t] + (-e - 1)
 * (include/shardplan/remap.hpp:27-29 encoding).  remap == NULL means the
 * identity placement (slot = row).  For each distinct (table, slot) — a
 * SEGMENT of the sorted list starting at position s, length L — the gradient
 * g = sum of grad_out[b, col_off[t] : +D] over its lookups, accumulated in
 * fp32 in the kernel's fixed tree (csrc/emb_bwd.cuh): pieces of 32 positions
 * from s, each summed in sorted order from +0.0f (L <= 32: g is that sum);
 * groups of 64 consecutive pieces added left to right (first piece as the
 * accumulator); g = the group sums left to right (first as the
 * accumulator).  Then
 *   opt 0 (row-wise SGD):  w[d] = w[d] - lr*g[d]
 *   opt 1 (exact row-wise Adagrad, FBGEMM semantics):
 *       s = sum_d g[d]^2   (per-lane then xor-butterfly order, see oracle.c)
 *       m = m + s / D;     mult = lr / (sqrtf(m) + eps);   w[d] = w[d] - mult*g[d]
 * All operations single-rounded fp32 (no contraction).  momentum[t] has H_t
 * slots (ignored for SGD). */
int or_emb_backward(uint32_t T, uint64_t B, const uint32_t* D,
                    const uint64_t* H, const uint64_t* col_off,
                    uint64_t grad_stride, const uint64_t* offsets,
                    const uint32_t* indices, const float* grad_out, int opt,
                    float lr, float eps, float* const* W,
                    float* const* momentum, const int32_t* const* remap,
                    const uint64_t* hbm_rows);

#ifdef __cplusplus
}
#endif
#endif
