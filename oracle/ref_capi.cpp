// TEST INFRASTRUCTURE ONLY.  extern "C" shim over the UNMODIFIED reference
// library (/root/reference/proj/core, compiled by oracle/Makefile into
// oracle/_ref/libshardplan_ref.so) so the Python tests, the golden-vector
// generator and bench.py's cpu_baseline leg can drive the reference through
// ctypes.  Nothing here is linked into, or called by, the product library.
//
// Every entry point returns 0 on success or a negative status; the error
// kinds mirror the reference exception taxonomy (inc/error.hpp:38-72):
//   -1 InvalidArgument  -2 ParseError  -3 InfeasibleError  -4 IoError
//   -5 std::out_of_range (profile's index_of.at, core/src/profiler.cpp:103)
//   -9 anything else

#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "shardplan/baselines.hpp"
#include "shardplan/milp.hpp"
#include "shardplan/profiler.hpp"
#include "shardplan/remap.hpp"
#include "shardplan/trace_io.hpp"
#include "shardplan/simulator.hpp"
#include "shardplan/workload.hpp"
#include "shardplan/zipf.hpp"

using namespace shardplan;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const InvalidArgument& e) {
    g_err = e.what();
    return -1;
  } catch (const ParseError& e) {
    g_err = e.what();
    return -2;
  } catch (const InfeasibleError& e) {
    g_err = e.what();
    return -3;
  } catch (const IoError& e) {
    g_err = e.what();
    return -4;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return -5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -9;
  }
}

std::vector<TableSpec> make_specs(uint32_t J, const uint32_t* table_id,
                                  const uint64_t* card,
                                  const uint64_t* hash_size,
                                  const uint32_t* dim,
                                  const uint32_t* elem_bytes) {
  std::vector<TableSpec> t(J);
  for (uint32_t j = 0; j < J; ++j)
    t[j] = TableSpec{table_id[j], card[j], hash_size[j], dim[j], elem_bytes[j]};
  return t;
}

struct TraceBox {
  Trace trace;
  GenStats gen;
  std::vector<uint64_t> raw_ids;  // only for refc_generate_raw_trace
};
struct StatsBox {
  std::vector<FeatureStats> stats;
};
struct PlanBox {
  ShardingPlan plan;
};
}  // namespace

extern "C" {

const char* refc_last_error() { return g_err.c_str(); }

int refc_hash_value(uint64_t raw, uint64_t hash_size, uint32_t* out) {
  return guarded([&] { *out = hash_value(raw, hash_size); });
}

int refc_mix64_batch(const uint64_t* in, uint64_t n, uint64_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = mix64(in[i]);
  return 0;
}

int refc_derive_stream(uint64_t master, uint64_t a, uint64_t b, uint64_t* out) {
  *out = derive_stream(master, a, b);
  return 0;
}

// ---------------------------------------------------------------- traces
int refc_generate_trace(uint32_t J, const uint32_t* table_id,
                        const uint64_t* card, const uint64_t* hash_size,
                        const uint32_t* dim, const uint32_t* elem_bytes,
                        const double* zipf, const double* mean_pool,
                        const double* coverage, const int* law,
                        uint64_t num_samples, uint64_t seed, int want_gen,
                        void** out) {
  return guarded([&] {
    auto specs_t = make_specs(J, table_id, card, hash_size, dim, elem_bytes);
    std::vector<WorkloadSpec> specs(J);
    for (uint32_t j = 0; j < J; ++j) {
      specs[j].table = specs_t[j];
      specs[j].gen = FeatureGenSpec{zipf[j], mean_pool[j], coverage[j],
                                    static_cast<PoolingLaw>(law[j])};
    }
    auto* box = new TraceBox;
    try {
      box->trace = generate_trace(specs, num_samples, seed,
                                  want_gen ? &box->gen : nullptr);
    } catch (...) {
      delete box;
      throw;
    }
    *out = box;
  });
}

// Raw (pre-hash) ids drawn exactly as generate_trace_range draws them
// (core/src/workload.cpp:198-217) but without the hash at :213, built only
// from the reference's public samplers.  Used to pin profile_raw parity:
// hash_value(raw) must equal the hashed trace bit for bit.
int refc_generate_raw_trace(uint32_t J, const uint32_t* table_id,
                            const uint64_t* card, const uint64_t* hash_size,
                            const uint32_t* dim, const uint32_t* elem_bytes,
                            const double* zipf, const double* mean_pool,
                            const double* coverage, const int* law,
                            uint64_t num_samples, uint64_t seed, void** out) {
  return guarded([&] {
    auto specs_t = make_specs(J, table_id, card, hash_size, dim, elem_bytes);
    auto* box = new TraceBox;
    box->trace.tables = specs_t;
    box->trace.num_samples = num_samples;
    std::vector<ZipfSampler> zs;
    std::vector<PoolingSampler> ps;
    for (uint32_t j = 0; j < J; ++j) {
      zs.emplace_back(card[j], zipf[j]);
      ps.emplace_back(static_cast<PoolingLaw>(law[j]),
                      coverage[j] > 0.0 ? mean_pool[j] : 1.0);
    }
    for (uint64_t s = 0; s < num_samples; ++s) {
      for (uint32_t j = 0; j < J; ++j) {
        SplitMix64 rng(derive_stream(seed, s, table_id[j]));
        if (coverage[j] <= 0.0 || rng.next_double() >= coverage[j]) continue;
        uint32_t k = ps[j](rng);
        Trace::Record rec;
        rec.sample = s;
        rec.table = table_id[j];
        rec.offset = box->raw_ids.size();
        rec.len = k;
        for (uint32_t i = 0; i < k; ++i) box->raw_ids.push_back(zs[j](rng));
        box->trace.records.push_back(rec);
      }
    }
    *out = box;
  });
}

int refc_trace_from_arrays(uint32_t J, const uint32_t* table_id,
                           const uint64_t* card, const uint64_t* hash_size,
                           const uint32_t* dim, const uint32_t* elem_bytes,
                           uint64_t num_samples, uint64_t R,
                           const uint64_t* rec_sample,
                           const uint32_t* rec_table,
                           const uint64_t* rec_offset, const uint32_t* rec_len,
                           uint64_t N, const uint32_t* ids, void** out) {
  return guarded([&] {
    auto* box = new TraceBox;
    box->trace.tables = make_specs(J, table_id, card, hash_size, dim, elem_bytes);
    box->trace.num_samples = num_samples;
    box->trace.records.resize(R);
    for (uint64_t r = 0; r < R; ++r)
      box->trace.records[r] = Trace::Record{rec_sample[r], rec_table[r],
                                            rec_offset[r], rec_len[r]};
    box->trace.ids.assign(ids, ids + N);
    *out = box;
  });
}

int refc_trace_sizes(void* h, uint64_t* R, uint64_t* N, uint64_t* N_raw) {
  auto* box = static_cast<TraceBox*>(h);
  *R = box->trace.records.size();
  *N = box->trace.ids.size();
  if (N_raw) *N_raw = box->raw_ids.size();
  return 0;
}

int refc_trace_copy(void* h, uint64_t* rec_sample, uint32_t* rec_table,
                    uint64_t* rec_offset, uint32_t* rec_len, uint32_t* ids,
                    uint64_t* raw_ids, uint64_t* distinct_raw) {
  auto* box = static_cast<TraceBox*>(h);
  const auto& t = box->trace;
  for (size_t r = 0; r < t.records.size(); ++r) {
    rec_sample[r] = t.records[r].sample;
    rec_table[r] = t.records[r].table;
    rec_offset[r] = t.records[r].offset;
    rec_len[r] = t.records[r].len;
  }
  if (ids && !t.ids.empty())
    std::memcpy(ids, t.ids.data(), t.ids.size() * sizeof(uint32_t));
  if (raw_ids && !box->raw_ids.empty())
    std::memcpy(raw_ids, box->raw_ids.data(), box->raw_ids.size() * 8);
  if (distinct_raw)
    for (size_t j = 0; j < box->gen.distinct_raw_ids.size(); ++j)
      distinct_raw[j] = box->gen.distinct_raw_ids[j];
  return 0;
}

void refc_trace_free(void* h) { delete static_cast<TraceBox*>(h); }

// core/src/trace_io.cpp:48-158
int refc_read_trace(const char* path, void** out) {
  return guarded([&] {
    auto* box = new TraceBox;
    try {
      box->trace = read_trace(path);
    } catch (...) {
      delete box;
      throw;
    }
    *out = box;
  });
}

int refc_write_trace(void* h, const char* path, const char* const* comments, uint32_t n) {
  return guarded([&] {
    std::vector<std::string> c(comments, comments + n);
    write_trace(static_cast<TraceBox*>(h)->trace, path, c);
  });
}

int refc_trace_meta(void* h, uint32_t* J, uint64_t* num_samples, uint32_t* table_id, uint64_t* card,
                    uint64_t* hash_size, uint32_t* dim, uint32_t* elem_bytes) {
  const auto& t = static_cast<TraceBox*>(h)->trace;
  *J = uint32_t(t.tables.size());
  *num_samples = t.num_samples;
  if (table_id)
    for (size_t j = 0; j < t.tables.size(); ++j) {
      table_id[j] = t.tables[j].table_id;
      card[j] = t.tables[j].cardinality;
      hash_size[j] = t.tables[j].hash_size;
      dim[j] = t.tables[j].dim;
      elem_bytes[j] = t.tables[j].elem_bytes;
    }
  return 0;
}

// ---------------------------------------------------------------- profile
int refc_profile(void* trace, double rate, uint64_t seed, void** out) {
  return guarded([&] {
    auto* box = new StatsBox;
    try {
      box->stats = profile(static_cast<TraceBox*>(trace)->trace, rate, seed);
    } catch (...) {
      delete box;
      throw;
    }
    *out = box;
  });
}

// Wall-clock seconds of one reference profile() call (cpu_baseline leg).
int refc_time_profile(void* trace, double rate, uint64_t seed, double* secs) {
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    auto st = profile(static_cast<TraceBox*>(trace)->trace, rate, seed);
    auto t1 = std::chrono::steady_clock::now();
    *secs = std::chrono::duration<double>(t1 - t0).count();
    if (st.empty()) *secs = -1;
  });
}

int refc_stats_new(uint32_t J, void** out) {
  auto* box = new StatsBox;
  box->stats.resize(J);
  *out = box;
  return 0;
}

int refc_stats_set(void* h, uint32_t j, uint32_t table_id, double coverage,
                   double avg_pooling, uint64_t distinct, uint64_t total,
                   const uint64_t* icdf101, const double* cdf,
                   const uint32_t* rows_by_rank) {
  auto& st = static_cast<StatsBox*>(h)->stats.at(j);
  st.table_id = table_id;
  st.coverage = coverage;
  st.avg_pooling = avg_pooling;
  st.distinct_rows_accessed = distinct;
  st.total_accesses = total;
  st.icdf_steps.assign(icdf101, icdf101 + 101);
  if (cdf) st.access_cdf.assign(cdf, cdf + distinct);
  if (rows_by_rank) st.rows_by_rank.assign(rows_by_rank, rows_by_rank + distinct);
  return 0;
}

int refc_stats_count(void* h) {
  return static_cast<int>(static_cast<StatsBox*>(h)->stats.size());
}

int refc_stats_scalars(void* h, uint32_t j, uint32_t* table_id, double* cov,
                       double* pool, uint64_t* distinct, uint64_t* total) {
  const auto& st = static_cast<StatsBox*>(h)->stats.at(j);
  *table_id = st.table_id;
  *cov = st.coverage;
  *pool = st.avg_pooling;
  *distinct = st.distinct_rows_accessed;
  *total = st.total_accesses;
  return 0;
}

int refc_stats_arrays(void* h, uint32_t j, uint64_t* icdf101, double* cdf,
                      uint32_t* rows_by_rank) {
  const auto& st = static_cast<StatsBox*>(h)->stats.at(j);
  if (icdf101) std::memcpy(icdf101, st.icdf_steps.data(), 101 * 8);
  if (cdf && !st.access_cdf.empty())
    std::memcpy(cdf, st.access_cdf.data(), st.access_cdf.size() * 8);
  if (rows_by_rank && !st.rows_by_rank.empty())
    std::memcpy(rows_by_rank, st.rows_by_rank.data(),
                st.rows_by_rank.size() * 4);
  return 0;
}

void refc_stats_free(void* h) { delete static_cast<StatsBox*>(h); }

int refc_build_icdf(const uint64_t* counts, uint64_t n, uint64_t* out101) {
  return guarded([&] {
    auto v = build_icdf(std::span<const uint64_t>(counts, n));
    std::memcpy(out101, v.data(), 101 * 8);
  });
}

int refc_hash_utilization(uint64_t distinct_rows, uint64_t hash_size,
                          uint64_t distinct_raw, double* sparsity,
                          double* collisions) {
  return guarded([&] {
    FeatureStats st;
    st.distinct_rows_accessed = distinct_rows;
    TableSpec spec{0, hash_size, hash_size, 4, 4};
    auto [s, c] = hash_utilization(st, spec, distinct_raw);
    *sparsity = s;
    *collisions = c;
  });
}

// ---------------------------------------------------------------- remap
int refc_build_remap(void* stats, uint32_t j, uint32_t table_id,
                     uint64_t hash_size, uint32_t dim, uint32_t elem_bytes,
                     uint64_t hbm_rows, int omit_unaccessed, int32_t* entries,
                     uint64_t* slow_rows_allocated) {
  return guarded([&] {
    const auto& st = static_cast<StatsBox*>(stats)->stats.at(j);
    PlanEntry e;
    e.table_id = table_id;
    e.hbm_rows = hbm_rows;
    TableSpec spec{table_id, hash_size, hash_size, dim, elem_bytes};
    RemapOptions opts;
    opts.omit_unaccessed = omit_unaccessed != 0;
    auto r = build_remap(e, st, spec, opts);
    std::memcpy(entries, r.entries.data(), r.entries.size() * 4);
    *slow_rows_allocated = r.slow_rows_allocated;
  });
}

// ---------------------------------------------------------------- SPRM files
int refc_write_remap(const char* path, uint32_t table_id, uint64_t hash_size, uint64_t hbm_rows,
                     const int32_t* entries) {
  return guarded([&] {
    RemapTable r;
    r.table_id = table_id;
    r.hash_size = hash_size;
    r.hbm_rows = hbm_rows;
    r.entries.assign(entries, entries + hash_size);
    write_remap(r, path);
  });
}

int refc_read_remap(const char* path, uint32_t* table_id, uint64_t* hash_size, uint64_t* hbm_rows,
                    int32_t* entries, uint64_t capacity, uint64_t* slow_rows_allocated) {
  return guarded([&] {
    RemapTable r = read_remap(path);
    *table_id = r.table_id;
    *hash_size = r.hash_size;
    *hbm_rows = r.hbm_rows;
    *slow_rows_allocated = r.slow_rows_allocated;
    if (r.entries.size() <= capacity) std::memcpy(entries, r.entries.data(), r.entries.size() * 4);
  });
}

// ---------------------------------------------------------------- simulate
int refc_simulate(void* trace, uint32_t n_entries, const uint32_t* e_table,
                  const uint32_t* e_gpu, const uint64_t* e_hbm_rows,
                  uint32_t n_remaps, const uint32_t* r_table,
                  const uint64_t* r_hash, const uint64_t* r_hbm,
                  const int32_t* const* r_entries, uint32_t num_gpus,
                  uint64_t sys_batch, uint64_t cap_hbm, uint64_t cap_dram,
                  double bw_hbm, double bw_uvm, uint64_t batch_size,
                  double* gpu_hbm, double* gpu_uvm, double* gpu_cost,
                  uint64_t* batches, uint64_t* total, double* agg5,
                  double* table_fast_fraction, double* secs) {
  return guarded([&] {
    ShardingPlan plan;
    plan.entries.resize(n_entries);
    for (uint32_t i = 0; i < n_entries; ++i) {
      plan.entries[i].table_id = e_table[i];
      plan.entries[i].gpu = e_gpu[i];
      plan.entries[i].hbm_rows = e_hbm_rows[i];
    }
    std::vector<RemapTable> remaps(n_remaps);
    for (uint32_t i = 0; i < n_remaps; ++i) {
      remaps[i].table_id = r_table[i];
      remaps[i].hash_size = r_hash[i];
      remaps[i].hbm_rows = r_hbm[i];
      remaps[i].entries.assign(r_entries[i], r_entries[i] + r_hash[i]);
    }
    SystemSpec sys{num_gpus, sys_batch, cap_hbm, cap_dram, bw_hbm, bw_uvm};
    const Trace& t = static_cast<TraceBox*>(trace)->trace;
    auto t0 = std::chrono::steady_clock::now();
    SimReport rep = simulate(t, plan, remaps, sys, batch_size);
    auto t1 = std::chrono::steady_clock::now();
    if (secs) *secs = std::chrono::duration<double>(t1 - t0).count();
    for (uint32_t g = 0; g < num_gpus; ++g) {
      gpu_hbm[g] = rep.gpus[g].hbm_accesses;
      gpu_uvm[g] = rep.gpus[g].uvm_accesses;
      gpu_cost[g] = rep.gpus[g].est_iter_cost;
    }
    *batches = rep.batches;
    *total = rep.total_accesses;
    agg5[0] = rep.min_cost;
    agg5[1] = rep.max_cost;
    agg5[2] = rep.mean_cost;
    agg5[3] = rep.stddev_cost;
    agg5[4] = rep.uvm_access_fraction;
    for (size_t j = 0; j < rep.table_fast_fraction.size(); ++j)
      table_fast_fraction[j] = rep.table_fast_fraction[j];
  });
}

// ---------------------------------------------------------------- planners
// kind: 0 milp solve, 1 greedy, 2 ldm; cost: 0 size, 1 lookup, 2 size-lookup
int refc_plan(void* trace, void* stats, int kind, int cost_kind,
              uint32_t num_gpus, uint64_t sys_batch, uint64_t cap_hbm,
              uint64_t cap_dram, double bw_hbm, double bw_uvm,
              uint32_t step_count, double time_limit, void** out) {
  return guarded([&] {
    const Trace& t = static_cast<TraceBox*>(trace)->trace;
    const auto& st = static_cast<StatsBox*>(stats)->stats;
    SystemSpec sys{num_gpus, sys_batch, cap_hbm, cap_dram, bw_hbm, bw_uvm};
    auto* box = new PlanBox;
    try {
      if (kind == 0) {
        auto inst = build_instance(st, t.tables, sys, {}, step_count);
        box->plan = solve(inst, time_limit);
      } else {
        std::vector<double> costs;
        for (size_t j = 0; j < t.tables.size(); ++j)
          costs.push_back(table_fixed_cost(t.tables[j], &st[j],
                                           static_cast<CostKind>(cost_kind)));
        box->plan = kind == 1 ? greedy_shard(costs, t.tables, st, sys)
                              : ldm_shard(costs, t.tables, st, sys);
      }
    } catch (...) {
      delete box;
      throw;
    }
    *out = box;
  });
}

int refc_plan_size(void* h, uint32_t* n, uint32_t* step_count,
                   double* objective) {
  const auto& p = static_cast<PlanBox*>(h)->plan;
  *n = static_cast<uint32_t>(p.entries.size());
  *step_count = p.step_count;
  *objective = p.objective;
  return 0;
}

int refc_plan_entries(void* h, uint32_t* table_id, uint32_t* gpu,
                      uint32_t* step, uint64_t* hbm_rows, double* pct,
                      uint64_t* mem_bytes) {
  const auto& p = static_cast<PlanBox*>(h)->plan;
  for (size_t i = 0; i < p.entries.size(); ++i) {
    table_id[i] = p.entries[i].table_id;
    gpu[i] = p.entries[i].gpu;
    step[i] = p.entries[i].step;
    hbm_rows[i] = p.entries[i].hbm_rows;
    pct[i] = p.entries[i].pct;
    mem_bytes[i] = p.entries[i].mem_bytes;
  }
  return 0;
}

void refc_plan_free(void* h) { delete static_cast<PlanBox*>(h); }

}  // extern "C"
