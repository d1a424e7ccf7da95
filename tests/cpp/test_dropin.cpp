// C++ drop-in parity: the reference's own calls, made twice — once into the
// unmodified reference library (shardplan::) and once through the GPU shim
// (shardplan::gpu::, include/shardplan_gpu.hpp) — must agree bit for bit.
// Mirrors the reference tests (tests/test_profiler.cpp, test_remap.cpp,
// test_simulator.cpp, test_workload.cpp) without doctest.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "shardplan/baselines.hpp"
#include "shardplan/milp.hpp"
#include "shardplan/trace_io.hpp"
#include "shardplan/workload.hpp"
#include "shardplan_gpu.hpp"

#include <cuda_runtime.h>

using namespace shardplan;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                          \
  do {                                                                    \
    if (c) ++g_pass;                                                      \
    else {                                                                \
      ++g_fail;                                                           \
      std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #c); \
    }                                                                     \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

static bool stats_equal(const std::vector<FeatureStats>& a, const std::vector<FeatureStats>& b) {
  if (a.size() != b.size()) return false;
  for (size_t j = 0; j < a.size(); ++j) {
    const auto &x = a[j], &y = b[j];
    if (x.table_id != y.table_id || !same(x.coverage, y.coverage) ||
        !same(x.avg_pooling, y.avg_pooling) ||
        x.distinct_rows_accessed != y.distinct_rows_accessed ||
        x.total_accesses != y.total_accesses || x.icdf_steps != y.icdf_steps ||
        x.rows_by_rank != y.rows_by_rank || x.access_cdf.size() != y.access_cdf.size())
      return false;
    for (size_t r = 0; r < x.access_cdf.size(); ++r)
      if (!same(x.access_cdf[r], y.access_cdf[r])) return false;
  }
  return true;
}

static Trace worked_example() {  // tests/test_profiler.cpp:30-49
  Trace t;
  t.tables = {TableSpec{0, 1000, 100, 4, 4}, TableSpec{1, 1000, 100, 4, 4}};
  t.num_samples = 3;
  auto add = [&](uint64_t s, uint32_t tab, std::initializer_list<uint32_t> ids) {
    t.records.push_back({s, tab, t.ids.size(), static_cast<uint32_t>(ids.size())});
    t.ids.insert(t.ids.end(), ids);
  };
  add(0, 0, {1, 5, 9, 15});
  add(0, 1, {2, 4, 8});
  add(1, 0, {5, 7, 9, 30});
  add(2, 0, {1, 5, 9});
  return t;
}

int main() {
  // hash_value goldens (tests/test_workload.cpp:50-57)
  CHECK(gpu::hash_value(42, 1ULL << 32) == 3564271138ULL);
  CHECK(gpu::hash_value(7, 1000) == 604);
  CHECK(throws<InvalidArgument>([] { gpu::hash_value(1, 0); }));
  SplitMix64 rng(99);
  for (int i = 0; i < 10000; ++i) {
    uint64_t raw = rng.next(), h = 1 + rng.next_below(0x7FFFFFFF);
    if (gpu::hash_value(raw, h) != hash_value(raw, h)) {
      CHECK(false);
      break;
    }
  }

  // Fig. 3 worked example (tests/test_profiler.cpp:53-62)
  {
    Trace t = worked_example();
    auto g = gpu::profile(t, 1.0, 0);
    CHECK(stats_equal(g, profile(t, 1.0, 0)));
    CHECK(g[0].total_accesses == 11 && g[0].distinct_rows_accessed == 6);
    CHECK(throws<InvalidArgument>([&] { gpu::profile(t, 0.0, 0); }));
    CHECK(throws<InvalidArgument>([&] { gpu::profile(Trace{}, 0.5, 0); }));
    CHECK(throws<InvalidArgument>([&] { gpu::profile(t, 1e-12, 0); }));
    Trace bad = t;
    bad.tables.pop_back();
    CHECK(throws<std::out_of_range>([&] { gpu::profile(bad, 1.0, 0); }));
  }

  // generated traces, full and sampled profiles
  std::vector<WorkloadSpec> specs(3);
  specs[0].table = {0, 4000, 3000, 16, 4};
  specs[0].gen = {1.3, 6.0, 0.9, PoolingLaw::kPoisson};
  specs[1].table = {1, 9000, 8000, 8, 4};
  specs[1].gen = {1.1, 3.0, 0.5, PoolingLaw::kLognormal};
  specs[2].table = {2, 2000, 1500, 32, 2};
  specs[2].gen = {0.9, 2.0, 1.0, PoolingLaw::kConstant};
  Trace t = generate_trace(specs, 20000, 5);
  for (auto [rate, seed] : {std::pair{1.0, 0ULL}, {0.01, 1ULL}, {0.37, 12ULL}})
    CHECK(stats_equal(gpu::profile(t, rate, seed), profile(t, rate, seed)));

  // build_icdf vs the reference on random vectors (tests/test_profiler.cpp:103-119)
  for (int trial = 0; trial < 200; ++trial) {
    size_t n = 1 + rng.next_below(1000);
    std::vector<uint64_t> c(n);
    bool any = false;
    for (auto& x : c) any |= (x = rng.next_below(100)) > 0;
    if (!any) c[0] = 1;
    if (gpu::build_icdf(c) != build_icdf(c)) {
      CHECK(false);
      break;
    }
  }
  CHECK(throws<InvalidArgument>([] { gpu::build_icdf(std::vector<uint64_t>(5, 0)); }));

  // plans -> remaps -> simulate (tests/test_simulator.cpp:40-58 pipeline)
  auto stats = profile(t, 1.0, 0);
  std::vector<TableSpec> tabs;
  for (auto& w : specs) tabs.push_back(w.table);
  SystemSpec sys{2, 256, 0, 1ULL << 30, 1.555e12, 1.6e10};
  uint64_t total = 0;
  for (auto& s : tabs) total += s.bytes();
  sys.cap_hbm_bytes = total / 3;
  auto inst = build_instance(stats, tabs, sys, {}, 20);
  std::vector<double> costs;
  for (size_t j = 0; j < tabs.size(); ++j)
    costs.push_back(table_fixed_cost(tabs[j], &stats[j], CostKind::kSize));
  for (const ShardingPlan& plan : {solve(inst, 2.0), greedy_shard(costs, tabs, stats, sys)}) {
    std::vector<RemapTable> ref_r, gpu_r;
    for (size_t j = 0; j < tabs.size(); ++j) {
      for (bool omit : {false, true}) {
        RemapOptions o;
        o.omit_unaccessed = omit;
        auto a = build_remap(plan.entries[j], stats[j], tabs[j], o);
        auto b = gpu::build_remap(plan.entries[j], stats[j], tabs[j], o);
        CHECK(a.entries == b.entries && a.slow_rows_allocated == b.slow_rows_allocated);
      }
      ref_r.push_back(build_remap(plan.entries[j], stats[j], tabs[j]));
      gpu_r.push_back(gpu::build_remap(plan.entries[j], stats[j], tabs[j]));
      for (uint64_t i = 0; i < tabs[j].hash_size; i += 97)
        CHECK(gpu::translate(gpu_r[j], i) == translate(ref_r[j], i));
      // SPRM files: each side reads what the other wrote (remap.cpp:118-176)
      const std::string pa = "/tmp/rs_dropin_a.sprm", pb = "/tmp/rs_dropin_b.sprm";
      write_remap(ref_r[j], pa);
      gpu::write_remap(gpu_r[j], pb);
      auto ra = gpu::read_remap(pa);
      auto rb = read_remap(pb);
      CHECK(ra.entries == rb.entries && ra.table_id == rb.table_id && ra.hbm_rows == rb.hbm_rows &&
            ra.hash_size == rb.hash_size && ra.slow_rows_allocated == rb.slow_rows_allocated);
      std::remove(pa.c_str());
      std::remove(pb.c_str());
    }
    for (uint64_t B : {256ULL, 1000ULL, 20000ULL}) {
      auto a = simulate(t, plan, ref_r, sys, B);
      auto b = gpu::simulate(t, plan, gpu_r, sys, B);
      bool eq = a.batches == b.batches && a.total_accesses == b.total_accesses &&
                same(a.min_cost, b.min_cost) && same(a.max_cost, b.max_cost) &&
                same(a.mean_cost, b.mean_cost) && same(a.stddev_cost, b.stddev_cost) &&
                same(a.uvm_access_fraction, b.uvm_access_fraction);
      for (size_t g = 0; g < a.gpus.size(); ++g)
        eq = eq && same(a.gpus[g].hbm_accesses, b.gpus[g].hbm_accesses) &&
             same(a.gpus[g].uvm_accesses, b.gpus[g].uvm_accesses) &&
             same(a.gpus[g].est_iter_cost, b.gpus[g].est_iter_cost);
      for (size_t j = 0; j < a.table_fast_fraction.size(); ++j)
        eq = eq && (same(a.table_fast_fraction[j], b.table_fast_fraction[j]) ||
                    (std::isnan(a.table_fast_fraction[j]) && std::isnan(b.table_fast_fraction[j])));
      CHECK(eq);
    }
    CHECK(throws<InvalidArgument>([&] { gpu::simulate(t, plan, gpu_r, sys, 1 << 30); }));
  }
  CHECK(throws<IoError>([] { gpu::read_remap("/nonexistent/x.sprm"); }));
  // trace files (core/src/trace_io.cpp): each side reads what the other wrote
  for (const char* ext : {".trace", ".trace.gz"}) {
    Trace t = generate_trace(specs, 3000, 21);
    const std::string pa = std::string("/tmp/rs_dropin_a") + ext, pb = std::string("/tmp/rs_dropin_b") + ext;
    write_trace(t, pa, {"ref"});
    gpu::write_trace(t, pb, {"ref"});
    Trace a = gpu::read_trace(pa), b = read_trace(pb);
    bool eq = a.num_samples == b.num_samples && a.ids == b.ids && a.records.size() == b.records.size() &&
              a.tables.size() == b.tables.size();
    for (size_t r = 0; eq && r < a.records.size(); ++r)
      eq = a.records[r].sample == b.records[r].sample && a.records[r].table == b.records[r].table &&
           a.records[r].offset == b.records[r].offset && a.records[r].len == b.records[r].len;
    CHECK(eq && a.ids == t.ids);
    std::remove(pa.c_str());
    std::remove(pb.c_str());
  }
  {
    FILE* f = std::fopen("/tmp/rs_dropin_bad.trace", "wb");
    std::fputs("#shardplan-trace v1 tables=1 samples=10\nT 0 100 100 4 4\nR zero 0 1\n", f);
    std::fclose(f);
    bool line3 = false;
    try {
      gpu::read_trace("/tmp/rs_dropin_bad.trace");
    } catch (const ParseError& e) {
      line3 = e.line() == 3 && std::string(e.what()) == "line 3: bad sample_id: 'zero'";
    }
    CHECK(line3);
    std::remove("/tmp/rs_dropin_bad.trace");
  }
  {
    FILE* f = std::fopen("/tmp/rs_dropin_bad.sprm", "wb");
    std::fwrite("SPRX", 1, 4, f);
    std::fclose(f);
    CHECK(throws<ParseError>([] { gpu::read_remap("/tmp/rs_dropin_bad.sprm"); }));
    std::remove("/tmp/rs_dropin_bad.sprm");
  }
  // TieredEmbeddingBag (the §8b operator) through the C++ shim: forward is
  // the in-order fp32 sum of each bag's rows (bit-exact vs a host loop over
  // read_rows), its hit counts are the remap's tier split, and the backward
  // (SGD, grad = pooled) moves exactly the rows the batch touched.
  {
    std::vector<TableSpec> ftabs;  // fp32 tables only
    std::vector<RemapTable> frem;
    std::vector<uint32_t> tid;
    for (size_t j = 0; j < tabs.size(); ++j)
      if (tabs[j].elem_bytes == 4) {
        ftabs.push_back(tabs[j]);
        PlanEntry pe{tabs[j].table_id, 0, 0, tabs[j].hash_size / 2, 0.0, 0};
        frem.push_back(gpu::build_remap(pe, stats[j], tabs[j]));
        tid.push_back(tabs[j].table_id);
      }
    const uint32_t T = static_cast<uint32_t>(ftabs.size());
    const uint64_t B = 256;
    // table-major CSR of the trace's first B samples
    std::vector<std::vector<std::vector<uint32_t>>> bags(T, std::vector<std::vector<uint32_t>>(B));
    for (const auto& r : t.records) {
      if (r.sample >= B) continue;
      for (uint32_t k = 0; k < T; ++k)
        if (t.tables[r.table].table_id == tid[k])
          for (uint32_t q = 0; q < r.len; ++q) bags[k][r.sample].push_back(t.ids[r.offset + q]);
    }
    std::vector<uint32_t> off{0}, idx;
    for (uint32_t k = 0; k < T; ++k)
      for (uint64_t b = 0; b < B; ++b) {
        idx.insert(idx.end(), bags[k][b].begin(), bags[k][b].end());
        off.push_back(static_cast<uint32_t>(idx.size()));
      }
    gpu::TieredEmbeddingBag op(ftabs, frem, B, std::max<size_t>(1, idx.size()));
    op.init_weights(7, 0.5f);
    uint32_t *d_off = nullptr, *d_idx = nullptr;
    float* d_out = nullptr;
    uint64_t* d_hits = nullptr;
    cudaMalloc(&d_off, off.size() * 4);
    cudaMalloc(&d_idx, std::max<size_t>(1, idx.size()) * 4);
    cudaMalloc(&d_out, B * op.total_dim() * 4);
    cudaMalloc(&d_hits, 2 * T * 8);
    cudaMemset(d_hits, 0, 2 * T * 8);
    cudaMemcpy(d_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_idx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
    std::vector<std::vector<float>> W(T);
    for (uint32_t k = 0; k < T; ++k) {
      std::vector<uint32_t> rows(ftabs[k].hash_size);
      for (uint32_t r = 0; r < rows.size(); ++r) rows[r] = r;
      W[k] = op.read_rows(k, rows, ftabs[k].dim);
    }
    op.forward(B, d_off, d_idx, d_out, d_hits);
    op.synchronize();  // the operator runs on the context's private stream
    std::vector<float> y(B * op.total_dim());
    std::vector<uint64_t> hits(2 * T);
    cudaMemcpy(y.data(), d_out, y.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hits.data(), d_hits, hits.size() * 8, cudaMemcpyDeviceToHost);
    bool fwd_ok = true, hits_ok = true;
    uint32_t col = 0;
    for (uint32_t k = 0; k < T; ++k) {
      const uint32_t D = ftabs[k].dim;
      uint64_t fast = 0, total = 0;
      for (uint64_t b = 0; b < B; ++b) {
        std::vector<float> acc(D, 0.0f);
        for (uint32_t row : bags[k][b]) {
          for (uint32_t d = 0; d < D; ++d) acc[d] = acc[d] + W[k][size_t(row) * D + d];
          fast += frem[k].entries[row] >= 0;
          ++total;
        }
        for (uint32_t d = 0; d < D; ++d) fwd_ok = fwd_ok && same(acc[d], y[b * op.total_dim() + col + d]);
      }
      hits_ok = hits_ok && hits[2 * k] == fast && hits[2 * k + 1] == total - fast;
      col += D;
    }
    CHECK(fwd_ok);
    CHECK(hits_ok);
    op.backward(B, d_off, d_idx, d_out, 0.1f);
    bool moved_ok = true;
    for (uint32_t k = 0; k < T; ++k) {
      std::vector<uint32_t> rows(ftabs[k].hash_size);
      for (uint32_t r = 0; r < rows.size(); ++r) rows[r] = r;
      auto w2 = op.read_rows(k, rows, ftabs[k].dim);
      std::vector<char> touched(rows.size(), 0);
      for (uint64_t b = 0; b < B; ++b)
        for (uint32_t row : bags[k][b]) touched[row] = 1;
      for (uint32_t r = 0; r < rows.size(); ++r) {
        bool changed = false;
        for (uint32_t d = 0; d < ftabs[k].dim; ++d)
          changed = changed || !same(w2[size_t(r) * ftabs[k].dim + d], W[k][size_t(r) * ftabs[k].dim + d]);
        if (!touched[r] && changed) moved_ok = false;
      }
    }
    CHECK(moved_ok);
    cudaFree(d_off);
    cudaFree(d_idx);
    cudaFree(d_out);
    cudaFree(d_hits);
  }
  std::printf("drop-in parity: %d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
