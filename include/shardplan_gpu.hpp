// shardplan_gpu.hpp — the reference's C++ value API over the C-ABI.
//
// A drop-in for callers of the reference library (tools/shardplan.cpp,
// tests/acceptance_main.cpp): include this next to the reference headers and
// call shardplan::gpu::profile / build_icdf / hash_utilization / hash_value /
// build_remap / translate / simulate with exactly the reference's argument
// types (plus the §8b extensions count_distinct_raw and TieredEmbeddingBag)
// types and semantics; errors rethrow the reference's exception types
// (include/shardplan/error.hpp:38-72, plus std::out_of_range for an unknown
// table in profile, core/src/profiler.cpp:103).
//
// Requires the reference's public headers on the include path (the types are
// the reference's own: shardplan::Trace, FeatureStats, PlanEntry, ...).
#pragma once

#include <cstdio>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "shardplan/profiler.hpp"
#include "shardplan/remap.hpp"
#include "shardplan/simulator.hpp"
#include "shardplan_gpu.h"

namespace shardplan::gpu {

[[noreturn]] inline void rethrow(int status) {
  const std::string m = rs_last_error();
  switch (status) {
    case RS_ERR_INVALID_ARGUMENT: throw InvalidArgument(m);
    case RS_ERR_PARSE: {
      // "line N: what" -> ParseError(what, N): same what(), and line() as the reference
      unsigned long long ln = 0;
      int used = 0;
      if (std::sscanf(m.c_str(), "line %llu: %n", &ln, &used) == 1 && used > 0 && ln > 0)
        throw ParseError(m.substr(size_t(used)), size_t(ln));
      throw ParseError(m);
    }
    case RS_ERR_INFEASIBLE: throw InfeasibleError(m);
    case RS_ERR_IO: throw IoError(m);
    case RS_ERR_OUT_OF_RANGE: throw std::out_of_range(m);
    default: throw Error(m);
  }
}

inline void check(int status) {
  if (status != RS_OK) rethrow(status);
}

/// One rs_context per device, on a private stream (calls are synchronous
/// from the caller's point of view, like the reference functions).
class Context {
 public:
  explicit Context(int device = 0) {
    check(rs_context_create(device, nullptr, RS_CTX_PRIVATE_STREAM, &ctx_));
  }
  ~Context() { rs_context_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  rs_context* get() const { return ctx_; }

  static Context& instance(int device = 0) {
    thread_local std::unique_ptr<Context> c;
    if (!c) c = std::make_unique<Context>(device);
    return *c;
  }

 private:
  rs_context* ctx_ = nullptr;
};

namespace detail {
// Structure-of-arrays view of a reference Trace (inc/workload.hpp:41-58).
struct TraceSoA {
  std::vector<rs_table_spec> specs;
  std::vector<uint64_t> sample, offset;
  std::vector<uint32_t> table, len;
  rs_trace view{};

  explicit TraceSoA(const Trace& t) {
    for (const auto& s : t.tables)
      specs.push_back({s.table_id, s.cardinality, s.hash_size, s.dim, s.elem_bytes});
    const size_t R = t.records.size();
    sample.resize(R);
    offset.resize(R);
    table.resize(R);
    len.resize(R);
    for (size_t r = 0; r < R; ++r) {
      sample[r] = t.records[r].sample;
      table[r] = t.records[r].table;
      offset[r] = t.records[r].offset;
      len[r] = t.records[r].len;
    }
    view.num_tables = static_cast<uint32_t>(specs.size());
    view.tables = specs.data();
    view.num_samples = t.num_samples;
    view.num_records = R;
    view.rec_sample = sample.data();
    view.rec_table = table.data();
    view.rec_offset = offset.data();
    view.rec_len = len.data();
    view.num_ids = t.ids.size();
    view.ids = t.ids.data();
    view.raw_ids = nullptr;
    view.location = RS_MEM_HOST;
  }
};
}  // namespace detail

/// inc/workload.hpp:28-31
inline uint32_t hash_value(uint64_t raw_id, uint64_t hash_size) {
  uint32_t out = 0;
  check(rs_hash_value(raw_id, hash_size, &out));
  return out;
}

/// include/shardplan/profiler.hpp:49-50 — K1 + K2 on the GPU.
inline std::vector<FeatureStats> profile(const Trace& trace, double sample_rate, uint64_t seed) {
  if (trace.num_samples < 1 || trace.tables.empty())  // profiler.cpp:62-63
    throw InvalidArgument("profile: trace is empty");
  detail::TraceSoA soa(trace);
  rs_profile* p = nullptr;
  check(rs_profile_run(Context::instance().get(), &soa.view, sample_rate, seed, &p));
  std::unique_ptr<rs_profile, int (*)(rs_profile*)> guard(p, rs_profile_destroy);
  uint32_t J = 0;
  check(rs_profile_num_tables(p, &J));
  std::vector<FeatureStats> out(J);
  for (uint32_t j = 0; j < J; ++j) {
    rs_feature_stats v{};
    check(rs_profile_get(p, j, &v));
    FeatureStats& s = out[j];
    s.table_id = v.table_id;
    s.coverage = v.coverage;
    s.avg_pooling = v.avg_pooling;
    s.distinct_rows_accessed = v.distinct_rows_accessed;
    s.total_accesses = v.total_accesses;
    s.icdf_steps.assign(v.icdf_steps, v.icdf_steps + kIcdfPercentSteps + 1);
    s.access_cdf.assign(v.access_cdf, v.access_cdf + v.distinct_rows_accessed);
    s.rows_by_rank.assign(v.rows_by_rank, v.rows_by_rank + v.distinct_rows_accessed);
  }
  return out;
}

/// include/shardplan/profiler.hpp:54
inline std::vector<uint64_t> build_icdf(std::span<const uint64_t> counts_per_row) {
  std::vector<uint64_t> out(kIcdfPercentSteps + 1);
  check(rs_build_icdf(Context::instance().get(), counts_per_row.data(), counts_per_row.size(),
                      RS_MEM_HOST, out.data()));
  return out;
}

/// include/shardplan/profiler.hpp:58-60
inline std::pair<double, double> hash_utilization(const FeatureStats& stats, const TableSpec& spec,
                                                  uint64_t distinct_raw_ids_seen) {
  std::pair<double, double> r;
  check(rs_hash_utilization(stats.distinct_rows_accessed, spec.hash_size, distinct_raw_ids_seen,
                            &r.first, &r.second));
  return r;
}

/// include/shardplan/remap.hpp:54-55 — K3 on the GPU.
inline RemapTable build_remap(const PlanEntry& entry, const FeatureStats& stats,
                              const TableSpec& spec, const RemapOptions& opts = {}) {
  if (stats.rows_by_rank.size() != stats.distinct_rows_accessed && spec.hash_size <= kMaxHashSize &&
      entry.hbm_rows <= spec.hash_size)  // remap.cpp:52-56 (after the bound checks)
    throw InvalidArgument(strfmt("table %u: stats lack row-level ranking (loaded from a stats "
                                 "file?); re-profile the trace",
                                 spec.table_id));
  RemapTable r;
  r.table_id = spec.table_id;
  r.hash_size = spec.hash_size;
  r.hbm_rows = entry.hbm_rows;
  r.entries.resize(spec.hash_size <= kMaxHashSize ? spec.hash_size : 0);
  check(rs_build_remap(Context::instance().get(), spec.table_id, spec.hash_size, entry.hbm_rows,
                       stats.rows_by_rank.data(), stats.distinct_rows_accessed, RS_MEM_HOST,
                       opts.omit_unaccessed ? 1 : 0, r.entries.data(), RS_MEM_HOST,
                       &r.slow_rows_allocated));
  return r;
}

/// core/src/remap.cpp:107-116 (host decode of the sign-bit encoding)
inline std::pair<Tier, uint64_t> translate(const RemapTable& remap, uint64_t original_index) {
  if (original_index >= remap.hash_size)
    throw InvalidArgument(strfmt("translate: index %llu out of range for table %u",
                                 (unsigned long long)original_index, remap.table_id));
  const int32_t v = remap.entries[original_index];
  if (v >= 0) return {Tier::kFast, static_cast<uint64_t>(v)};
  return {Tier::kSlow, static_cast<uint64_t>(-(int64_t)v - 1)};
}

/// include/shardplan/remap.hpp:62 — SPRM file, byte-identical to the reference's writer.
inline void write_remap(const RemapTable& remap, const std::string& path) {
  if (remap.entries.size() != remap.hash_size)
    throw InvalidArgument(strfmt("write_remap: table %u has %zu entries for hash_size %llu",
                                 remap.table_id, remap.entries.size(),
                                 (unsigned long long)remap.hash_size));
  check(rs_remap_write(nullptr, path.c_str(), remap.table_id, remap.hash_size, remap.hbm_rows,
                       remap.entries.empty() ? nullptr : remap.entries.data(), RS_MEM_HOST));
}

/// include/shardplan/remap.hpp:63 — reference errors (IoError / ParseError) preserved.
inline RemapTable read_remap(const std::string& path) {
  RemapTable r;
  uint32_t tid = 0;
  uint64_t H = 0, hbm = 0;
  check(rs_remap_read_header(path.c_str(), &tid, &H, &hbm));
  r.table_id = tid;
  r.hash_size = H;
  r.hbm_rows = hbm;
  r.entries.resize(H);
  int32_t dummy = 0;
  check(rs_remap_read(nullptr, path.c_str(), H ? r.entries.data() : &dummy, RS_MEM_HOST, H,
                      &r.slow_rows_allocated));
  return r;
}

/// A trace file loaded on the GPU (rs_trace_file): the records and ids stay in
/// device memory; view() is an rs_trace for rs_profile_run / rs_simulate.
class TraceFile {
 public:
  explicit TraceFile(const std::string& path, uint64_t chunk_bytes = 0) {
    check(rs_trace_read(Context::instance().get(), path.c_str(), chunk_bytes, &f_));
  }
  ~TraceFile() { rs_trace_file_destroy(f_); }
  TraceFile(const TraceFile&) = delete;
  TraceFile& operator=(const TraceFile&) = delete;
  rs_trace view() const {
    rs_trace v{};
    check(rs_trace_file_view(f_, &v));
    return v;
  }
  /// The reference's value type (records and ids copied to the host).
  Trace to_host() const {
    const rs_trace v = view();
    Trace t;
    for (uint32_t j = 0; j < v.num_tables; ++j) {
      const rs_table_spec& s = v.tables[j];
      t.tables.push_back(TableSpec{s.table_id, s.cardinality, s.hash_size, s.dim, s.elem_bytes});
    }
    t.num_samples = v.num_samples;
    std::vector<uint64_t> smp(v.num_records), off(v.num_records);
    std::vector<uint32_t> tab(v.num_records), len(v.num_records);
    t.ids.resize(v.num_ids);
    check(rs_trace_file_export(Context::instance().get(), f_, smp.data(), tab.data(), off.data(), len.data(),
                               t.ids.data(), RS_MEM_HOST));
    t.records.resize(v.num_records);
    for (size_t r = 0; r < t.records.size(); ++r) t.records[r] = Trace::Record{smp[r], tab[r], off[r], len[r]};
    return t;
  }

 private:
  rs_trace_file* f_ = nullptr;
};

/// include/shardplan/trace_io.hpp:35 — parsed on the GPU, same errors.
inline Trace read_trace(const std::string& path) { return TraceFile(path).to_host(); }

/// include/shardplan/trace_io.hpp:32-33 — byte-identical to the reference writer.
inline void write_trace(const Trace& trace, const std::string& path,
                        const std::vector<std::string>& comments = {}) {
  detail::TraceSoA soa(trace);
  std::vector<const char*> cs;
  for (const auto& c : comments) cs.push_back(c.c_str());
  check(rs_trace_write(Context::instance().get(), &soa.view, path.c_str(), cs.empty() ? nullptr : cs.data(),
                       static_cast<uint32_t>(cs.size())));
}

/// include/shardplan/simulator.hpp:45-47 — tier counts on the GPU.
inline SimReport simulate(const Trace& trace, const ShardingPlan& plan,
                          const std::vector<RemapTable>& remaps, const SystemSpec& system,
                          uint64_t batch_size) {
  detail::TraceSoA soa(trace);
  std::vector<rs_plan_entry> ents;
  for (const auto& e : plan.entries)
    ents.push_back({e.table_id, e.gpu, e.step, e.hbm_rows, e.pct, e.mem_bytes});
  std::vector<rs_remap_view> rv;
  for (const auto& r : remaps)
    rv.push_back({r.table_id, r.hash_size, r.hbm_rows, r.entries.data(), RS_MEM_HOST});
  rs_system_spec sys{system.num_gpus, system.batch_size, system.cap_hbm_bytes,
                     system.cap_dram_bytes, system.bw_hbm, system.bw_uvm};
  SimReport rep;
  const uint32_t M = system.num_gpus;
  std::vector<double> gh(M ? M : 1), gu(M ? M : 1), gc(M ? M : 1);
  rep.table_fast_fraction.resize(trace.tables.size());
  rs_sim_report out{};
  out.gpu_hbm_accesses = gh.data();
  out.gpu_uvm_accesses = gu.data();
  out.gpu_est_iter_cost = gc.data();
  out.table_fast_fraction = rep.table_fast_fraction.data();
  check(rs_simulate(Context::instance().get(), &soa.view, static_cast<uint32_t>(ents.size()),
                    ents.data(), static_cast<uint32_t>(rv.size()), rv.data(), &sys, batch_size,
                    &out));
  rep.gpus.resize(M);
  for (uint32_t g = 0; g < M; ++g) rep.gpus[g] = {gh[g], gu[g], gc[g]};
  rep.batches = out.batches;
  rep.total_accesses = out.total_accesses;
  rep.min_cost = out.min_cost;
  rep.max_cost = out.max_cost;
  rep.mean_cost = out.mean_cost;
  rep.stddev_cost = out.stddev_cost;
  rep.uvm_access_fraction = out.uvm_access_fraction;
  return rep;
}

/// SURVEY §8b extension: GenStats.distinct_raw_ids (core/src/workload.cpp:195-223)
/// of a trace carrying raw ids, counted on the GPU (one value per trace table).
inline std::vector<uint64_t> count_distinct_raw(const Trace& trace, const std::vector<uint64_t>& raw_ids) {
  detail::TraceSoA soa(trace);
  soa.view.ids = nullptr;
  soa.view.raw_ids = raw_ids.data();
  soa.view.num_ids = raw_ids.size();
  std::vector<uint64_t> out(trace.tables.size());
  check(rs_count_distinct_raw(Context::instance().get(), &soa.view, out.data()));
  return out;
}

/// The tiered EmbeddingBag serving a sharding plan (the paper ran
/// FBGEMM): rows the remap sends to the fast tier live in HBM,
/// the others in pinned host memory (fp32 or fp16 rows, fp32 arithmetic).  forward = sum-pool (an empty bag pools
/// to 0) with per-table fast/slow hit counts equal to
/// simulate()'s accounting; backward = deterministic row-wise SGD or exact
/// row-wise Adagrad.  Batches are table-major CSR in DEVICE memory
/// (offsets[T*B+1], indices = original rows); the pooled output is
/// [B, sum dim] fp32.  Calls are stream-ordered on the object's context.
class TieredEmbeddingBag {
 public:
  enum class Optimizer { kSgd = RS_OPT_SGD, kRowwiseAdagrad = RS_OPT_ROWWISE_ADAGRAD };

  TieredEmbeddingBag(const std::vector<TableSpec>& specs, const std::vector<RemapTable>& remaps,
                     uint64_t max_batch, uint64_t max_lookups, Optimizer opt = Optimizer::kSgd,
                     float eps = 1e-8f, Context& ctx = Context::instance())
      : ctx_(ctx) {
    if (specs.size() != remaps.size()) throw InvalidArgument("TieredEmbeddingBag: one remap per table");
    std::vector<rs_emb_table> tabs;
    for (size_t i = 0; i < specs.size(); ++i) {
      const auto& s = specs[i];
      const auto& r = remaps[i];
      // elem_bytes 2 or 4 (inc/types.hpp:50-52; validated by rs_emb_create);
      // an omit_unaccessed remap (inc/remap.hpp:43-48) backs only its
      // slow_rows_allocated prefix and the other slow rows pool as zeros
      const uint64_t slow = s.hash_size - r.hbm_rows;
      const int unbacked = r.slow_rows_allocated < slow ? 1 : 0;
      tabs.push_back({s.table_id, s.hash_size, s.dim, r.entries.data(), RS_MEM_HOST, r.hbm_rows,
                      unbacked ? r.slow_rows_allocated : slow, s.elem_bytes, unbacked});
      total_dim_ += s.dim;
    }
    check(rs_emb_create(ctx_.get(), static_cast<uint32_t>(tabs.size()), tabs.data(), max_batch, max_lookups,
                        static_cast<int>(opt), eps, &e_));
  }
  ~TieredEmbeddingBag() {
    if (e_) rs_emb_destroy(e_);
  }
  TieredEmbeddingBag(const TieredEmbeddingBag&) = delete;
  TieredEmbeddingBag& operator=(const TieredEmbeddingBag&) = delete;

  uint32_t total_dim() const { return total_dim_; }
  void init_weights(uint64_t seed, float scale) { check(rs_emb_init_weights(e_, seed, scale)); }
  void forward(uint64_t batch, const uint32_t* d_offsets, const uint32_t* d_indices, float* d_pooled,
               uint64_t* d_hit_counts = nullptr) {
    check(rs_emb_forward(e_, batch, d_offsets, d_indices, d_pooled, d_hit_counts));
  }
  void backward(uint64_t batch, const uint32_t* d_offsets, const uint32_t* d_indices, const float* d_grad,
                float lr) {
    check(rs_emb_backward(e_, batch, d_offsets, d_indices, d_grad, lr));
  }
  /// Slow-row staging (copy engines, one batch ahead): enable once, then
  /// prefetch(batch k+1) before batch k's forward.
  void enable_uvm_cache(uint32_t nslots) { check(rs_emb_enable_uvm_cache(e_, nslots)); }
  void prefetch(uint64_t batch, const uint32_t* d_offsets, const uint32_t* d_indices) {
    check(rs_emb_prefetch(e_, batch, d_offsets, d_indices));
  }
  void flush() { check(rs_emb_flush(e_)); }
  /// Rows by ORIGINAL id (and their Adagrad state) into host vectors.
  std::vector<float> read_rows(uint32_t table, const std::vector<uint32_t>& rows, uint32_t dim,
                               std::vector<float>* momentum = nullptr) {
    std::vector<float> out(rows.size() * dim);
    std::vector<float> m(rows.size());
    check(rs_emb_read_rows(e_, table, rows.data(), rows.size(), out.data(), m.data()));
    if (momentum) *momentum = std::move(m);
    return out;
  }
  /// Blocks until the object's queued work is done (before reading its
  /// outputs from another stream).
  void synchronize() { check(rs_context_synchronize(ctx_.get())); }
  rs_emb* handle() const { return e_; }

 private:
  Context& ctx_;
  rs_emb* e_ = nullptr;
  uint32_t total_dim_ = 0;
};

}  // namespace shardplan::gpu
