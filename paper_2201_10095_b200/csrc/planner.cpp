// Host planner: the cost model, the whole-table baselines (greedy, LDM) and
// the RecShard solver, with placements identical to the reference's.
//
// Restated from (paths relative to /root/reference/proj/core/):
//   cost model      src/plan.cpp:25-63        (table_cost, rows_at_step,
//                                              recompute_plan_costs)
//   baselines       src/baselines.cpp:44-292  (table_fixed_cost, greedy_shard,
//                                              ldm_shard)
//   instance        src/milp.cpp:20-60        (build_instance validation)
//   solver          src/milp_solve.cpp:22-709 (solve)
//
// The plan is a pure function of (specs, stats, system): every floating-point
// sum and comparison below is done in the reference's order with the
// reference's tolerances, so the placements match bit for bit.  What changes
// is the runtime: the solver's local search
// (milp_solve.cpp:536-602) re-solves only the two GPUs a candidate move
// touches (the others keep their allocation from the current assignment),
// evaluates its candidate moves on a pool of host threads, and then scans
// the results in the reference's order with its `better_than` tie-breaks;
// the per-GPU greedy allocation merges pre-sorted segment lists instead of
// sorting, and the assignment search keeps each GPU's relaxation segments
// sorted incrementally.  None of that charges the deterministic node budget
// differently, so budget trips (and therefore plans) are unchanged.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/shardplan_gpu.h"

namespace rs {
namespace plan {

struct PlanError : std::runtime_error {
  int status;
  PlanError(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};

static std::string fmt(const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}
[[noreturn]] static void invalid(const std::string& m) { throw PlanError(RS_ERR_INVALID_ARGUMENT, m); }
[[noreturn]] static void infeasible(const std::string& m) { throw PlanError(RS_ERR_INFEASIBLE, m); }

// ------------------------------------------------------------------ model
struct Table {
  rs_table_spec spec;
  double coverage, avg_pooling;
  const uint64_t* icdf;  // 101
  uint64_t bytes() const { return spec.hash_size * spec.dim * spec.elem_bytes; }
};

struct Abl {
  bool pooling = true, coverage = true;
};

// inc/types.hpp:97-110
static void validate_system(const rs_system_spec& s) {
  if (s.num_gpus < 1) invalid("system: num_gpus must be >= 1");
  if (s.batch_size < 1) invalid("system: batch_size must be >= 1");
  if (s.cap_hbm_bytes < 1) invalid("system: cap_hbm_bytes must be positive");
  if (s.cap_dram_bytes < 1) invalid("system: cap_dram_bytes must be positive");
  if (!(s.bw_hbm > 0.0) || !(s.bw_uvm > 0.0)) invalid("system: bandwidths must be positive");
  if (!(s.bw_hbm > s.bw_uvm)) invalid("system: bw_hbm must exceed bw_uvm");
}

// inc/types.hpp:40-55
static void validate_spec(const rs_table_spec& t) {
  if (t.hash_size < 1) invalid(fmt("table %u: hash_size must be >= 1", t.table_id));
  if (t.hash_size > 0x7FFFFFFFULL)
    invalid(fmt("table %u: hash_size %llu exceeds the 2^31-1 row limit imposed by the 4-byte remap encoding",
                t.table_id, (unsigned long long)t.hash_size));
  if (t.dim < 1) invalid(fmt("table %u: dim must be >= 1", t.table_id));
  if (t.elem_bytes != 2 && t.elem_bytes != 4) invalid(fmt("table %u: elem_bytes must be 2 or 4", t.table_id));
  if (t.cardinality < 1) invalid(fmt("table %u: cardinality must be >= 1", t.table_id));
}

// src/plan.cpp:25-33 — seconds of forward lookups at fast-tier fraction pct
static double table_cost(const Table& t, double pct, const rs_system_spec& sys, const Abl& abl) {
  if (!(pct >= 0.0 && pct <= 1.0)) invalid("table_cost: pct must be in [0, 1]");
  const double pool = abl.pooling ? t.avg_pooling : 1.0;
  const double demand = pool * t.spec.dim * t.spec.elem_bytes * static_cast<double>(sys.batch_size);
  return demand * (pct / sys.bw_hbm + (1.0 - pct) / sys.bw_uvm);
}

// src/plan.cpp:35-43
static uint64_t rows_at_step(const uint64_t* icdf, uint32_t step, uint32_t step_count) {
  if (step > step_count) invalid("rows_at_step: step exceeds step_count");
  const uint64_t pidx = (uint64_t(step) * 100 + step_count - 1) / step_count;
  return icdf[pidx];
}

struct Plan {
  std::vector<rs_plan_entry> entries;
  std::vector<double> gpu_cost;
  double objective = 0.0, lower_bound = 0.0;
  bool proved = false;
};

// src/plan.cpp:45-62 (entries are aligned with `tabs`)
static void recompute_costs(Plan& p, const std::vector<Table>& tabs, const rs_system_spec& sys, const Abl& abl) {
  p.gpu_cost.assign(sys.num_gpus, 0.0);
  for (size_t j = 0; j < p.entries.size(); ++j) {
    const rs_plan_entry& e = p.entries[j];
    const double w = abl.coverage ? tabs[j].coverage : 1.0;
    p.gpu_cost.at(e.gpu) += w * table_cost(tabs[j], e.pct, sys, abl);
  }
  p.objective = 0.0;
  for (double c : p.gpu_cost) p.objective = std::max(p.objective, c);
}

// src/milp.cpp:20-56 (the instance is aligned (spec, stats) pairs already)
static void validate_instance(const std::vector<Table>& tabs, const rs_system_spec& sys, uint32_t step_count) {
  if (tabs.empty()) invalid("build_instance: no tables");
  if (step_count < 1) invalid("build_instance: step_count must be >= 1");
  validate_system(sys);
  for (const Table& t : tabs) {
    validate_spec(t.spec);
    if (t.icdf[100] > t.spec.hash_size)
      invalid(fmt("build_instance: table %u icdf exceeds hash_size", t.spec.table_id));
  }
}

// ------------------------------------------------------------------ baselines
// src/baselines.cpp:44-67
static double fixed_cost(const rs_table_spec& s, const double* avg_pooling, int kind) {
  switch (kind) {
    case RS_COST_SIZE:
      return static_cast<double>(s.hash_size) * s.dim;
    case RS_COST_LOOKUP:
      if (!avg_pooling) invalid("lookup cost needs feature stats");
      return *avg_pooling * s.dim;
    case RS_COST_SIZE_LOOKUP: {
      if (!avg_pooling) invalid("size-lookup cost needs feature stats");
      double lg = std::log10(static_cast<double>(s.hash_size));
      if (lg < 0.0) {
        std::fprintf(stderr, "warning: table %u hash_size %llu < 10, clamping log10 factor to 0\n", s.table_id,
                     (unsigned long long)s.hash_size);
        lg = 0.0;
      }
      return *avg_pooling * s.dim * lg;
    }
  }
  invalid("unknown cost function");
}

// Tables by descending cost, ties by ascending table id (baselines.cpp:74-90).
static std::vector<uint32_t> cost_order(const std::vector<double>& costs, const std::vector<Table>& tabs) {
  if (costs.size() != tabs.size()) invalid("baseline: costs and specs differ in length");
  if (tabs.empty()) invalid("baseline: no tables");
  for (double c : costs)
    if (!(c >= 0.0) || !std::isfinite(c)) invalid("baseline: costs must be finite and >= 0");
  std::vector<uint32_t> o(tabs.size());
  std::iota(o.begin(), o.end(), 0u);
  std::sort(o.begin(), o.end(), [&](uint32_t a, uint32_t b) {
    if (costs[a] != costs[b]) return costs[a] > costs[b];
    return tabs[a].spec.table_id < tabs[b].spec.table_id;
  });
  return o;
}

static void check_aggregate(const std::vector<Table>& tabs, const rs_system_spec& sys) {
  uint64_t total = 0;
  for (const Table& t : tabs) total += t.bytes();
  const uint64_t agg = uint64_t(sys.num_gpus) * (sys.cap_hbm_bytes + sys.cap_dram_bytes);
  if (total > agg)
    infeasible(fmt("total table bytes %llu exceed aggregate capacity %llu", (unsigned long long)total,
                   (unsigned long long)agg));
}

// Whole-table plan on the 1-step grid (baselines.cpp:92-117).
static Plan whole_table_plan(const std::vector<Table>& tabs, const rs_system_spec& sys,
                             const std::vector<uint32_t>& gpu_of, const std::vector<char>& in_hbm) {
  validate_instance(tabs, sys, 100);
  Plan p;
  p.entries.resize(tabs.size());
  for (size_t j = 0; j < tabs.size(); ++j) {
    rs_plan_entry& e = p.entries[j];
    e.table_id = tabs[j].spec.table_id;
    e.gpu = gpu_of[j];
    e.step = in_hbm[j] ? 1 : 0;
    e.pct = in_hbm[j] ? 1.0 : 0.0;
    e.hbm_rows = in_hbm[j] ? tabs[j].spec.hash_size : 0;
    e.mem_bytes = e.hbm_rows * tabs[j].spec.dim * tabs[j].spec.elem_bytes;
  }
  recompute_costs(p, tabs, sys, Abl{});
  return p;
}

// src/baselines.cpp:136-203
static Plan greedy(const std::vector<double>& costs, const std::vector<Table>& tabs, const rs_system_spec& sys) {
  validate_system(sys);
  check_aggregate(tabs, sys);
  const std::vector<uint32_t> order = cost_order(costs, tabs);
  const uint32_t M = sys.num_gpus;
  std::vector<uint32_t> gpu_of(tabs.size(), 0);
  std::vector<char> in_hbm(tabs.size(), 0);
  std::vector<double> hbm_sum(M, 0.0), tot_sum(M, 0.0);
  std::vector<uint64_t> hbm_used(M, 0), uvm_used(M, 0);
  const double uvm_scale = sys.bw_hbm / sys.bw_uvm;
  bool hbm_phase = true;
  for (size_t pos = 0; pos < order.size(); ++pos) {
    const uint32_t j = order[pos];
    const uint64_t bytes = tabs[j].bytes();
    const double c = costs[j];
    if (hbm_phase) {
      uint32_t pick = UINT32_MAX;
      if (pos < M) {  // one of the first M tables per GPU
        if (hbm_used[pos] + bytes <= sys.cap_hbm_bytes) pick = uint32_t(pos);
      } else {
        double best = 0.0;
        for (uint32_t g = 0; g < M; ++g) {
          if (hbm_used[g] + bytes > sys.cap_hbm_bytes) continue;
          if (pick == UINT32_MAX || hbm_sum[g] < best) pick = g, best = hbm_sum[g];
        }
      }
      if (pick != UINT32_MAX) {
        gpu_of[j] = pick;
        in_hbm[j] = 1;
        hbm_used[pick] += bytes;
        hbm_sum[pick] += c;
        tot_sum[pick] += c;
        continue;
      }
      hbm_phase = false;
    }
    uint32_t pick = UINT32_MAX;
    double best = 0.0;
    for (uint32_t g = 0; g < M; ++g) {
      if (uvm_used[g] + bytes > sys.cap_dram_bytes) continue;
      if (pick == UINT32_MAX || tot_sum[g] < best) pick = g, best = tot_sum[g];
    }
    if (pick == UINT32_MAX)
      infeasible(fmt("greedy: table %u (%llu bytes) fits no GPU's slow tier", tabs[j].spec.table_id,
                     (unsigned long long)bytes));
    gpu_of[j] = pick;
    uvm_used[pick] += bytes;
    tot_sum[pick] += c * uvm_scale;
  }
  return whole_table_plan(tabs, sys, gpu_of, in_hbm);
}

// src/baselines.cpp:205-292 — multiway largest differencing
static Plan ldm(const std::vector<double>& costs, const std::vector<Table>& tabs, const rs_system_spec& sys) {
  validate_system(sys);
  check_aggregate(tabs, sys);
  const std::vector<uint32_t> order = cost_order(costs, tabs);
  const uint32_t M = sys.num_gpus;
  struct Part {
    double sum = 0.0;
    std::vector<uint32_t> tabs;
  };
  struct Tuple {
    std::vector<Part> parts;  // descending sum
    uint64_t seq = 0;
    double spread() const { return parts.front().sum - parts.back().sum; }
  };
  // largest spread first; equal spreads: the earliest-created tuple first
  auto lower = [](const Tuple& a, const Tuple& b) {
    if (a.spread() != b.spread()) return a.spread() < b.spread();
    return a.seq > b.seq;
  };
  std::priority_queue<Tuple, std::vector<Tuple>, decltype(lower)> q(lower);
  uint64_t seq = 0;
  for (uint32_t j : order) {
    Tuple t;
    t.parts.resize(M);
    t.parts[0].sum = costs[j];
    t.parts[0].tabs = {j};
    t.seq = seq++;
    q.push(std::move(t));
  }
  while (q.size() > 1) {
    Tuple a = q.top();
    q.pop();
    Tuple b = q.top();
    q.pop();
    Tuple m;
    m.parts.resize(M);
    for (uint32_t s = 0; s < M; ++s) {
      const Part& hi = a.parts[s];
      const Part& lo = b.parts[M - 1 - s];
      m.parts[s].sum = hi.sum + lo.sum;
      m.parts[s].tabs = hi.tabs;
      m.parts[s].tabs.insert(m.parts[s].tabs.end(), lo.tabs.begin(), lo.tabs.end());
    }
    std::stable_sort(m.parts.begin(), m.parts.end(), [](const Part& x, const Part& y) { return x.sum > y.sum; });
    m.seq = seq++;
    q.push(std::move(m));
  }
  const Tuple fin = q.top();
  std::vector<uint32_t> gpu_of(tabs.size(), 0);
  std::vector<char> in_hbm(tabs.size(), 0);
  for (uint32_t g = 0; g < M; ++g) {
    std::vector<uint32_t> mine = fin.parts[g].tabs;
    std::sort(mine.begin(), mine.end(), [&](uint32_t a, uint32_t b) {
      if (costs[a] != costs[b]) return costs[a] > costs[b];
      return tabs[a].spec.table_id < tabs[b].spec.table_id;
    });
    uint64_t hu = 0, uu = 0;
    for (uint32_t j : mine) {
      const uint64_t bytes = tabs[j].bytes();
      gpu_of[j] = g;
      if (hu + bytes <= sys.cap_hbm_bytes) {
        in_hbm[j] = 1;
        hu += bytes;
      } else if (uu + bytes <= sys.cap_dram_bytes) {
        uu += bytes;
      } else {
        infeasible(fmt("ldm: table %u (%llu bytes) fits neither tier of gpu %u", tabs[j].spec.table_id,
                       (unsigned long long)bytes, g));
      }
    }
  }
  return whole_table_plan(tabs, sys, gpu_of, in_hbm);
}

// ------------------------------------------------------------------ solver
constexpr double kRelTol = 1e-12;
constexpr double kHuge = std::numeric_limits<double>::max();

static inline double tol3(double a, double b) { return kRelTol * std::max({1.0, std::fabs(a), std::fabs(b)}); }
// milp_solve.cpp:27-34
static inline bool definitely_less(double a, double b) {
  if (b >= kHuge) return a < b;
  return a < b - tol3(a, b);
}
static inline bool roughly_equal(double a, double b) { return std::fabs(a - b) <= tol3(a, b); }

// A hull segment of one table: step `from` -> `to` saves dsave for dmem
// fast-tier bytes (milp_solve.cpp:38-44).
struct Seg {
  double rate = 0.0;
  uint64_t dmem = 0;
  double dsave = 0.0;
  uint32_t from = 0, to = 0;
};

// Per-table step grid and its concave hull (milp_solve.cpp:48-61, 88-153).
struct Curve {
  uint64_t emb = 0;
  std::vector<uint64_t> mem;
  std::vector<double> cost;
  uint32_t max_step = 0;
  std::vector<Seg> segs;  // rate descending (hull order)
  double cost0 = 0.0, solo_min = 0.0, impact = 0.0;
  uint64_t max_mem = 0, min_uvm = 0;
};

static Curve make_curve(const Table& t, const rs_system_spec& sys, const Abl& abl, uint32_t steps,
                        uint64_t cap_hbm) {
  Curve c;
  c.emb = t.bytes();
  const double w = abl.coverage ? t.coverage : 1.0;
  const uint64_t row_bytes = uint64_t(t.spec.dim) * t.spec.elem_bytes;
  c.mem.resize(steps + 1);
  c.cost.resize(steps + 1);
  for (uint32_t i = 0; i <= steps; ++i) {
    c.mem[i] = rows_at_step(t.icdf, i, steps) * row_bytes;
    c.cost[i] = w * table_cost(t, static_cast<double>(i) / steps, sys, abl);
  }
  c.cost0 = c.cost[0];
  while (c.max_step < steps && c.mem[c.max_step + 1] <= cap_hbm) ++c.max_step;
  c.max_mem = c.mem[c.max_step];
  c.min_uvm = c.emb - c.max_mem;
  c.solo_min = c.cost[0];
  for (uint32_t i = 1; i <= c.max_step; ++i) c.solo_min = std::min(c.solo_min, c.cost[i]);
  c.impact = c.cost[0];
  // distinct-mem points (a run of equal mem keeps its last step), then the
  // upper concave hull of (mem, saving)
  std::vector<uint32_t> pts;
  for (uint32_t i = 0; i <= c.max_step; ++i) {
    if (!pts.empty() && c.mem[pts.back()] == c.mem[i]) pts.back() = i;
    else pts.push_back(i);
  }
  auto save = [&](uint32_t i) { return c.cost0 - c.cost[i]; };
  std::vector<uint32_t> hull;
  for (uint32_t i : pts) {
    while (hull.size() >= 2) {
      const uint32_t a = hull[hull.size() - 2], b = hull.back();
      const double lhs = (save(b) - save(a)) * static_cast<double>(c.mem[i] - c.mem[a]);
      const double rhs = (save(i) - save(a)) * static_cast<double>(c.mem[b] - c.mem[a]);
      if (lhs <= rhs) hull.pop_back();
      else break;
    }
    hull.push_back(i);
  }
  for (size_t k = 1; k < hull.size(); ++k) {
    Seg s;
    s.from = hull[k - 1];
    s.to = hull[k];
    s.dmem = c.mem[s.to] - c.mem[s.from];
    s.dsave = save(s.to) - save(s.from);
    if (s.dmem == 0 || s.dsave <= 0.0) continue;
    s.rate = s.dsave / static_cast<double>(s.dmem);
    c.segs.push_back(s);
  }
  return c;
}

// A segment of a member list: (rate, member position, index within the
// table).  Every ordering the reference builds with stable_sort over
// (member order, segment order) by descending rate is this key.
struct SegRef {
  const Seg* seg;
  uint32_t pos;  // member position (local index)
  uint32_t k;
};
static inline bool seg_before(const SegRef& x, const SegRef& y) {
  if (x.seg->rate != y.seg->rate) return x.seg->rate > y.seg->rate;
  if (x.pos != y.pos) return x.pos < y.pos;
  return x.k < y.k;
}

struct Ctx {
  uint32_t J = 0, M = 0, steps = 0;
  uint64_t cap_hbm = 0, cap_dram = 0;
  std::vector<Curve> curves;
  double root_lb = 0.0;
  uint64_t budget = UINT64_MAX;
  bool budget_hit = false;
  // milp_solve.cpp:76-85 — the deterministic work budget
  bool charge(uint64_t n) {
    if (budget == UINT64_MAX) return true;
    if (budget < n) {
      budget = 0;
      budget_hit = true;
      return false;
    }
    budget -= n;
    return true;
  }
};

// Continuous relaxation over segments already in (rate desc, pos, k) order
// (milp_solve.cpp:157-175 after its sort).
static double relaxed_save(const std::vector<SegRef>& sorted, uint64_t cap) {
  double save = 0.0;
  uint64_t left = cap;
  for (const SegRef& r : sorted) {
    if (left == 0) break;
    if (r.seg->dmem <= left) {
      save += r.seg->dsave;
      left -= r.seg->dmem;
    } else {
      save += r.seg->rate * static_cast<double>(left);
      left = 0;
    }
  }
  return save;
}

struct Alloc {
  bool feasible = false;
  double cost = 0.0;
  uint64_t mem = 0;
  std::vector<uint32_t> steps;  // aligned with the member list
};

// The member list's segments in (rate desc, pos, k) order: a k-way merge of
// the tables' hull lists (each already rate-descending).
static void sorted_segs(const Ctx& ctx, const uint32_t* members, size_t n, std::vector<SegRef>& out) {
  out.clear();
  for (size_t l = 0; l < n; ++l) {
    const auto& s = ctx.curves[members[l]].segs;
    for (uint32_t k = 0; k < s.size(); ++k) out.push_back({&s[k], uint32_t(l), k});
  }
  std::sort(out.begin(), out.end(), seg_before);
}

// milp_solve.cpp:189-229 — greedy step allocation with lo <= mem <= hi.
static Alloc greedy_alloc_sorted(const Ctx& ctx, const uint32_t* members, size_t n, const std::vector<SegRef>& refs,
                                 uint64_t hi, uint64_t lo) {
  Alloc a;
  a.steps.assign(n, 0);
  for (size_t l = 0; l < n; ++l) a.cost += ctx.curves[members[l]].cost0;
  for (const SegRef& r : refs) {
    if (a.steps[r.pos] != r.seg->from) continue;
    if (a.mem + r.seg->dmem > hi) continue;
    a.steps[r.pos] = r.seg->to;
    a.mem += r.seg->dmem;
    a.cost -= r.seg->dsave;
  }
  for (size_t l = 0; l < n; ++l) {
    const Curve& c = ctx.curves[members[l]];
    while (a.steps[l] < c.max_step) {
      const uint64_t dm = c.mem[a.steps[l] + 1] - c.mem[a.steps[l]];
      if (a.mem + dm > hi) break;
      a.cost -= c.cost[a.steps[l]] - c.cost[a.steps[l] + 1];
      a.mem += dm;
      ++a.steps[l];
    }
  }
  a.feasible = a.mem >= lo && a.mem <= hi;
  a.cost = std::max(a.cost, 0.0);
  return a;
}

static uint64_t gpu_lo(const Ctx& ctx, const uint32_t* members, size_t n) {
  uint64_t emb = 0;
  for (size_t l = 0; l < n; ++l) emb += ctx.curves[members[l]].emb;
  return emb > ctx.cap_dram ? emb - ctx.cap_dram : 0;
}

static Alloc greedy_alloc(const Ctx& ctx, const std::vector<uint32_t>& members, uint64_t hi, uint64_t lo) {
  thread_local std::vector<SegRef> refs;
  sorted_segs(ctx, members.data(), members.size(), refs);
  return greedy_alloc_sorted(ctx, members.data(), members.size(), refs, hi, lo);
}

// milp_solve.cpp:231-327 — exact multiple-choice knapsack (DFS, lexicographic
// first optimum), bounded by the continuous relaxation of the suffix.
class Mckp {
 public:
  Mckp(Ctx& ctx, const std::vector<uint32_t>& members, uint64_t hi, uint64_t lo)
      : ctx_(ctx), mem_(members), hi_(hi), lo_(lo) {
    const size_t n = members.size();
    suf_cost0_.assign(n + 1, 0.0);
    suf_max_.assign(n + 1, 0);
    for (size_t d = n; d-- > 0;) {
      const Curve& c = ctx.curves[members[d]];
      suf_cost0_[d] = suf_cost0_[d + 1] + c.cost0;
      suf_max_[d] = suf_max_[d + 1] + c.max_mem;
    }
    sorted_segs(ctx, members.data(), n, segs_);
  }
  Alloc run(double cutoff) {
    best_ = Alloc{};
    best_.cost = cutoff;
    cur_.assign(mem_.size(), 0);
    dfs(0, 0, 0.0);
    return best_;
  }

 private:
  double suffix_bound(size_t d, uint64_t cap) const {
    double save = 0.0;
    uint64_t left = cap;
    for (const SegRef& r : segs_) {
      if (left == 0) break;
      if (r.pos < d) continue;
      if (r.seg->dmem <= left) {
        save += r.seg->dsave;
        left -= r.seg->dmem;
      } else {
        save += r.seg->rate * static_cast<double>(left);
        left = 0;
      }
    }
    return suf_cost0_[d] - save;
  }
  void dfs(size_t d, uint64_t mem, double cost) {
    if (!ctx_.charge(2)) return;
    if (d == mem_.size()) {
      if (mem >= lo_ && definitely_less(cost, best_.cost)) {
        best_.feasible = true;
        best_.cost = cost;
        best_.mem = mem;
        best_.steps = cur_;
      }
      return;
    }
    if (mem + suf_max_[d] < lo_) return;
    const double lb = cost + suffix_bound(d, hi_ - mem);
    if (!definitely_less(lb, best_.cost)) return;
    const Curve& c = ctx_.curves[mem_[d]];
    for (uint32_t i = 0; i <= c.max_step; ++i) {
      if (mem + c.mem[i] > hi_) break;
      if (ctx_.budget_hit) return;
      cur_[d] = i;
      dfs(d + 1, mem + c.mem[i], cost + c.cost[i]);
    }
  }
  Ctx& ctx_;
  const std::vector<uint32_t>& mem_;
  uint64_t hi_, lo_;
  std::vector<double> suf_cost0_;
  std::vector<uint64_t> suf_max_;
  std::vector<SegRef> segs_;
  Alloc best_;
  std::vector<uint32_t> cur_;
};

enum class Mode { kGreedy, kExactLex, kExactWarm };

// milp_solve.cpp:337-352
static Alloc solve_gpu(Ctx& ctx, const std::vector<uint32_t>& members, Mode mode) {
  const uint64_t lo = gpu_lo(ctx, members.data(), members.size());
  if (mode == Mode::kGreedy) return greedy_alloc(ctx, members, ctx.cap_hbm, lo);
  if (mode == Mode::kExactLex) {
    Mckp k(ctx, members, ctx.cap_hbm, lo);
    return k.run(kHuge);
  }
  Alloc g = greedy_alloc(ctx, members, ctx.cap_hbm, lo);
  Mckp k(ctx, members, ctx.cap_hbm, lo);
  Alloc e = k.run(g.feasible ? g.cost : kHuge);
  return e.feasible ? e : g;
}

struct Cand {
  bool valid = false;
  double objective = 0.0, total = 0.0;
  std::vector<uint32_t> gpu, step;
};

// milp_solve.cpp:368-377 — relabel GPUs by first use in table order
static void canonicalize(Cand& c, uint32_t M) {
  std::vector<uint32_t> map(M, UINT32_MAX);
  uint32_t next = 0;
  for (uint32_t& g : c.gpu) {
    if (map[g] == UINT32_MAX) map[g] = next++;
    g = map[g];
  }
}

// milp_solve.cpp:379-391
static bool better_than(const Cand& a, const Cand& b) {
  if (!b.valid) return a.valid;
  if (!a.valid) return false;
  if (definitely_less(a.objective, b.objective)) return true;
  if (definitely_less(b.objective, a.objective)) return false;
  if (definitely_less(a.total, b.total)) return true;
  if (definitely_less(b.total, a.total)) return false;
  if (a.gpu != b.gpu) return a.gpu < b.gpu;
  return a.step < b.step;
}

static std::vector<std::vector<uint32_t>> members_of(const Ctx& ctx, const std::vector<uint32_t>& gpu_of) {
  std::vector<std::vector<uint32_t>> m(ctx.M);
  for (uint32_t t = 0; t < ctx.J; ++t) m[gpu_of[t]].push_back(t);
  return m;
}

// milp_solve.cpp:393-417.  `given` (optional) supplies allocations for GPUs
// whose member list is unchanged (their Alloc is a pure function of it).
static Cand evaluate(Ctx& ctx, const std::vector<uint32_t>& gpu_of, Mode mode,
                     const std::vector<const Alloc*>* given = nullptr,
                     const std::vector<std::vector<uint32_t>>* members_in = nullptr) {
  Cand c;
  std::vector<std::vector<uint32_t>> own;
  const auto& members = members_in ? *members_in : (own = members_of(ctx, gpu_of));
  c.gpu = gpu_of;
  c.step.assign(ctx.J, 0);
  double objective = 0.0, total = 0.0;
  for (uint32_t m = 0; m < ctx.M; ++m) {
    if (members[m].empty()) continue;
    Alloc local;
    const Alloc* a = given ? (*given)[m] : nullptr;
    if (!a) {
      local = solve_gpu(ctx, members[m], mode);
      a = &local;
    }
    if (!a->feasible) return c;
    for (size_t l = 0; l < members[m].size(); ++l) c.step[members[m][l]] = a->steps[l];
    objective = std::max(objective, a->cost);
    total += a->cost;
  }
  c.objective = objective;
  c.total = total;
  c.valid = true;
  canonicalize(c, ctx.M);
  return c;
}

// milp_solve.cpp:423-513 — assignment branch and bound.  Each GPU's
// relaxation segments are kept in (rate desc, member position, k) order as
// tables are pushed and popped, instead of being re-sorted at every node.
class AssignSearch {
 public:
  AssignSearch(Ctx& ctx, bool exact)
      : ctx_(ctx), exact_(exact), members_(ctx.M), sorted_(ctx.M), lb_(ctx.M, 0.0), min_uvm_(ctx.M, 0),
        gpu_of_(ctx.J, UINT32_MAX) {
    order_.resize(ctx.J);
    std::iota(order_.begin(), order_.end(), 0u);
    std::stable_sort(order_.begin(), order_.end(),
                     [&](uint32_t a, uint32_t b) { return ctx_.curves[a].impact > ctx_.curves[b].impact; });
    solo_suffix_.assign(ctx.J + 1, 0.0);
    for (size_t d = ctx.J; d-- > 0;)
      solo_suffix_[d] = std::max(solo_suffix_[d + 1], ctx_.curves[order_[d]].solo_min);
  }
  void run(Cand& inc) {
    inc_ = &inc;
    dfs(0, 0);
  }

 private:
  double relaxed_lb(uint32_t m) const {
    double base = 0.0;
    for (uint32_t t : members_[m]) base += ctx_.curves[t].cost0;
    return base - relaxed_save(sorted_[m], ctx_.cap_hbm);
  }
  // t appended at position p of GPU m: merge its hull (already rate-desc,
  // k ascending) behind equal-rate segments of earlier positions
  void push_segs(uint32_t m, uint32_t t, uint32_t p) {
    auto& v = sorted_[m];
    const auto& s = ctx_.curves[t].segs;
    std::vector<SegRef> add(s.size());
    for (uint32_t k = 0; k < s.size(); ++k) add[k] = {&s[k], p, k};
    const size_t mid = v.size();
    v.insert(v.end(), add.begin(), add.end());
    std::inplace_merge(v.begin(), v.begin() + mid, v.end(), seg_before);
  }
  void pop_segs(uint32_t m, uint32_t p) {
    auto& v = sorted_[m];
    v.erase(std::remove_if(v.begin(), v.end(), [p](const SegRef& r) { return r.pos == p; }), v.end());
  }
  void dfs(uint32_t depth, uint32_t used) {
    if (ctx_.budget_hit) return;
    if (depth == ctx_.J) {
      if (!ctx_.charge(20 + 4ULL * ctx_.J)) return;
      Cand c = evaluate(ctx_, gpu_of_, exact_ ? Mode::kExactLex : Mode::kGreedy);
      if (c.valid && better_than(c, *inc_)) *inc_ = c;
      return;
    }
    const uint32_t t = order_[depth];
    const uint32_t open = std::min<uint32_t>(ctx_.M, used + 1);
    for (uint32_t g = 0; g < open; ++g) {
      if (!ctx_.charge(4 + members_[g].size())) return;
      if (min_uvm_[g] + ctx_.curves[t].min_uvm > ctx_.cap_dram) continue;
      const uint32_t p = uint32_t(members_[g].size());
      members_[g].push_back(t);
      push_segs(g, t, p);
      gpu_of_[t] = g;
      min_uvm_[g] += ctx_.curves[t].min_uvm;
      const double saved = lb_[g];
      lb_[g] = relaxed_lb(g);
      double node_lb = std::max(ctx_.root_lb, solo_suffix_[depth + 1]);
      for (uint32_t m = 0; m < ctx_.M; ++m) node_lb = std::max(node_lb, lb_[m]);
      const bool prune = inc_->valid && !definitely_less(node_lb, inc_->objective) &&
                         !roughly_equal(node_lb, inc_->objective);
      if (!prune) dfs(depth + 1, std::max(used, g + 1));
      lb_[g] = saved;
      min_uvm_[g] -= ctx_.curves[t].min_uvm;
      gpu_of_[t] = UINT32_MAX;
      pop_segs(g, p);
      members_[g].pop_back();
      if (ctx_.budget_hit) return;
    }
  }
  Ctx& ctx_;
  bool exact_;
  std::vector<uint32_t> order_;
  std::vector<double> solo_suffix_;
  std::vector<std::vector<uint32_t>> members_;
  std::vector<std::vector<SegRef>> sorted_;
  std::vector<double> lb_;
  std::vector<uint64_t> min_uvm_;
  std::vector<uint32_t> gpu_of_;
  Cand* inc_ = nullptr;
};

// milp_solve.cpp:519-554 — longest-processing-time seed
static Cand lpt_seed(Ctx& ctx) {
  std::vector<uint32_t> order(ctx.J);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t a, uint32_t b) { return ctx.curves[a].impact > ctx.curves[b].impact; });
  std::vector<std::vector<uint32_t>> members(ctx.M);
  std::vector<double> cost(ctx.M, 0.0);
  std::vector<uint32_t> gpu_of(ctx.J, 0);
  for (uint32_t t : order) {
    double best_peak = kHuge, best_cost = 0.0;
    uint32_t best_g = 0;
    bool placed = false;
    for (uint32_t g = 0; g < ctx.M; ++g) {
      auto& mem = members[g];
      mem.insert(std::lower_bound(mem.begin(), mem.end(), t), t);
      const Alloc a = greedy_alloc(ctx, mem, ctx.cap_hbm, gpu_lo(ctx, mem.data(), mem.size()));
      mem.erase(std::find(mem.begin(), mem.end(), t));
      if (!a.feasible) continue;
      double peak = a.cost;
      for (uint32_t o = 0; o < ctx.M; ++o)
        if (o != g) peak = std::max(peak, cost[o]);
      if (definitely_less(peak, best_peak)) {
        best_peak = peak;
        best_g = g;
        best_cost = a.cost;
        placed = true;
      }
    }
    auto& mem = members[best_g];
    mem.insert(std::lower_bound(mem.begin(), mem.end(), t), t);
    if (placed) cost[best_g] = best_cost;
    gpu_of[t] = best_g;
  }
  return evaluate(ctx, gpu_of, Mode::kGreedy);
}

// Runs f(i) for i in [0, n) on `threads` threads (dynamic chunks).
template <class F>
static void parallel_for(size_t n, unsigned threads, F&& f) {
  if (threads <= 1 || n < 2) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
  };
  std::vector<std::thread> pool;
  const unsigned T = unsigned(std::min<size_t>(threads, n));
  for (unsigned k = 1; k < T; ++k) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
}

// milp_solve.cpp:556-602 — move / swap local search on the peak GPU.  A
// candidate changes two GPUs' member lists; the rest keep this round's
// allocation.  Candidates are evaluated in parallel, then reduced in the
// reference's scan order with its acceptance test and tie-breaks.
static Cand local_search(Ctx& ctx, Cand start, unsigned threads) {
  if (!start.valid) return start;
  Cand cur = start;
  for (int round = 0; round < 200; ++round) {
    const auto members = members_of(ctx, cur.gpu);
    std::vector<Alloc> base(ctx.M);
    std::vector<double> cost(ctx.M, 0.0);
    for (uint32_t g = 0; g < ctx.M; ++g) {
      if (members[g].empty()) continue;
      base[g] = greedy_alloc(ctx, members[g], ctx.cap_hbm, gpu_lo(ctx, members[g].data(), members[g].size()));
      cost[g] = base[g].feasible ? base[g].cost : kHuge;
    }
    uint32_t b = 0;
    for (uint32_t g = 1; g < ctx.M; ++g)
      if (cost[g] > cost[b]) b = g;
    auto improves = [&](const Cand& c) {
      return definitely_less(c.objective, cur.objective) ||
             (roughly_equal(c.objective, cur.objective) && definitely_less(c.total, cur.total));
    };
    // candidate k: (t -> g) moves, then (t -> g, u -> b) swaps if no move helps
    struct Move {
      uint32_t t, g, u;  // u == UINT32_MAX: plain move
    };
    auto run_phase = [&](const std::vector<Move>& moves) {
      std::vector<Cand> out(moves.size());
      parallel_for(moves.size(), threads, [&](size_t i) {
        const Move& mv = moves[i];
        std::vector<uint32_t> gpu_of = cur.gpu;
        gpu_of[mv.t] = mv.g;
        if (mv.u != UINT32_MAX) gpu_of[mv.u] = b;
        std::vector<std::vector<uint32_t>> mem = members;
        auto& mb = mem[b];
        mb.erase(std::find(mb.begin(), mb.end(), mv.t));
        auto& mg = mem[mv.g];
        mg.insert(std::lower_bound(mg.begin(), mg.end(), mv.t), mv.t);
        if (mv.u != UINT32_MAX) {
          mg.erase(std::find(mg.begin(), mg.end(), mv.u));
          mb.insert(std::lower_bound(mb.begin(), mb.end(), mv.u), mv.u);
        }
        std::vector<const Alloc*> given(ctx.M, nullptr);
        for (uint32_t m = 0; m < ctx.M; ++m)
          if (m != b && m != mv.g) given[m] = &base[m];
        Cand c = evaluate(ctx, gpu_of, Mode::kGreedy, &given, &mem);
        if (c.valid && improves(c)) out[i] = std::move(c);
      });
      Cand best;
      for (Cand& c : out)
        if (c.valid && better_than(c, best)) best = std::move(c);
      return best;
    };
    std::vector<Move> moves;
    for (uint32_t t : members[b])
      for (uint32_t g = 0; g < ctx.M; ++g)
        if (g != b) moves.push_back({t, g, UINT32_MAX});
    Cand best = run_phase(moves);
    if (!best.valid) {
      moves.clear();
      for (uint32_t t : members[b])
        for (uint32_t g = 0; g < ctx.M; ++g) {
          if (g == b) continue;
          for (uint32_t u : members[g]) moves.push_back({t, g, u});
        }
      best = run_phase(moves);
    }
    if (!best.valid) break;
    cur = std::move(best);
  }
  return cur;
}

// milp_solve.cpp:606-612
static Cand polish(Ctx& ctx, const Cand& c) {
  if (!c.valid) return c;
  Cand out = evaluate(ctx, c.gpu, Mode::kExactWarm);
  if (out.valid && better_than(out, c)) return out;
  return c;
}

// milp_solve.cpp:614-629
static double pooled_root_lb(const Ctx& ctx) {
  std::vector<SegRef> all;
  double base = 0.0, solo = 0.0;
  for (uint32_t t = 0; t < ctx.J; ++t) {
    const Curve& c = ctx.curves[t];
    base += c.cost0;
    solo = std::max(solo, c.solo_min);
    for (uint32_t k = 0; k < c.segs.size(); ++k) all.push_back({&c.segs[k], t, k});
  }
  std::sort(all.begin(), all.end(), seg_before);
  const double pooled = (base - relaxed_save(all, ctx.cap_hbm * uint64_t{ctx.M})) / ctx.M;
  return std::max(pooled, solo);
}

// milp_solve.cpp:633-709
static Plan solve(const std::vector<Table>& tabs, const rs_system_spec& sys, uint32_t step_count, const Abl& abl,
                  double time_limit, unsigned threads) {
  validate_instance(tabs, sys, step_count);
  uint64_t total = 0;
  for (const Table& t : tabs) total += t.bytes();
  const uint64_t agg = uint64_t{sys.num_gpus} * (sys.cap_hbm_bytes + sys.cap_dram_bytes);
  if (total > agg)
    infeasible(fmt("total table bytes %llu exceed aggregate capacity M*(cap_hbm+cap_dram) = %llu "
                   "(fast/slow capacity constraints)",
                   (unsigned long long)total, (unsigned long long)agg));
  Ctx ctx;
  ctx.J = uint32_t(tabs.size());
  ctx.M = sys.num_gpus;
  ctx.steps = step_count;
  ctx.cap_hbm = sys.cap_hbm_bytes;
  ctx.cap_dram = sys.cap_dram_bytes;
  ctx.curves.reserve(tabs.size());
  for (const Table& t : tabs) ctx.curves.push_back(make_curve(t, sys, abl, step_count, sys.cap_hbm_bytes));
  for (size_t j = 0; j < tabs.size(); ++j)
    if (ctx.curves[j].min_uvm > ctx.cap_dram)
      infeasible(fmt("table %u needs %llu slow-tier bytes even at its maximal fast-tier split, exceeding "
                     "cap_dram %llu (slow-tier capacity constraint)",
                     tabs[j].spec.table_id, (unsigned long long)ctx.curves[j].min_uvm,
                     (unsigned long long)ctx.cap_dram));
  const bool exact = ctx.J <= 10 && ctx.M <= 3 && ctx.steps <= 12;
  if (exact) ctx.budget = UINT64_MAX;
  else if (!std::isfinite(time_limit)) ctx.budget = 20ULL * 1000 * 1000;
  else ctx.budget = static_cast<uint64_t>(std::min(std::max(1.0, time_limit) * 350000.0, 4e9));
  ctx.root_lb = pooled_root_lb(ctx);
  Cand inc;
  if (!exact) inc = polish(ctx, local_search(ctx, lpt_seed(ctx), threads));
  AssignSearch search(ctx, exact);
  search.run(inc);
  if (!exact && inc.valid) inc = polish(ctx, inc);
  if (!inc.valid) {
    if (!ctx.budget_hit)
      infeasible("no feasible placement exists: per-GPU fast/slow capacity constraints cannot all be met");
    infeasible("no feasible placement found within the search budget; raise the time limit or capacities");
  }
  Plan p;
  p.proved = !ctx.budget_hit;
  p.entries.resize(tabs.size());
  for (uint32_t t = 0; t < ctx.J; ++t) {
    rs_plan_entry& e = p.entries[t];
    e.table_id = tabs[t].spec.table_id;
    e.gpu = inc.gpu[t];
    e.step = inc.step[t];
    e.pct = static_cast<double>(e.step) / step_count;
    e.hbm_rows = rows_at_step(tabs[t].icdf, e.step, step_count);
    e.mem_bytes = e.hbm_rows * tabs[t].spec.dim * tabs[t].spec.elem_bytes;
  }
  recompute_costs(p, tabs, sys, abl);
  p.lower_bound = p.proved ? p.objective : ctx.root_lb;
  return p;
}

static std::vector<Table> tables_of(uint32_t J, const rs_plan_table* in) {
  if (J && !in) invalid("planner: tables is NULL");
  std::vector<Table> v(J);
  for (uint32_t j = 0; j < J; ++j) {
    if (!in[j].icdf_steps) invalid("planner: icdf_steps is NULL");
    v[j] = Table{in[j].spec, in[j].coverage, in[j].avg_pooling, in[j].icdf_steps};
  }
  return v;
}

static void emit(const Plan& p, rs_plan_entry* out, double* gpu_cost, uint32_t M, rs_plan_summary* sum) {
  if (out) std::copy(p.entries.begin(), p.entries.end(), out);
  if (gpu_cost) std::copy(p.gpu_cost.begin(), p.gpu_cost.begin() + std::min<size_t>(M, p.gpu_cost.size()), gpu_cost);
  if (sum) {
    sum->objective = p.objective;
    sum->lower_bound = p.lower_bound;
    sum->proved_optimal = p.proved ? 1 : 0;
  }
}

}  // namespace plan
}  // namespace rs

namespace {
thread_local std::string g_plan_err;
template <class F>
int plan_guard(F&& f) {
  try {
    f();
    return RS_OK;
  } catch (const rs::plan::PlanError& e) {
    g_plan_err = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_plan_err = "host allocation failed";
    return RS_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_plan_err = e.what();
    return RS_ERR_INTERNAL;
  }
}
}  // namespace

extern "C" {

const char* rs_plan_last_error(void) { return g_plan_err.c_str(); }

int rs_table_fixed_cost(const rs_table_spec* spec, const double* avg_pooling, int kind, double* out) {
  return plan_guard([&] {
    if (!spec || !out) rs::plan::invalid("rs_table_fixed_cost: NULL argument");
    *out = rs::plan::fixed_cost(*spec, avg_pooling, kind);
  });
}

int rs_plan_greedy(uint32_t J, const rs_plan_table* tables, const double* costs, const rs_system_spec* sys,
                   rs_plan_entry* out, double* gpu_cost, rs_plan_summary* summary) {
  return plan_guard([&] {
    if (!sys || (J && !costs)) rs::plan::invalid("rs_plan_greedy: NULL argument");
    auto tabs = rs::plan::tables_of(J, tables);
    auto p = rs::plan::greedy(std::vector<double>(costs, costs + J), tabs, *sys);
    rs::plan::emit(p, out, gpu_cost, sys->num_gpus, summary);
  });
}

int rs_plan_ldm(uint32_t J, const rs_plan_table* tables, const double* costs, const rs_system_spec* sys,
                rs_plan_entry* out, double* gpu_cost, rs_plan_summary* summary) {
  return plan_guard([&] {
    if (!sys || (J && !costs)) rs::plan::invalid("rs_plan_ldm: NULL argument");
    auto tabs = rs::plan::tables_of(J, tables);
    auto p = rs::plan::ldm(std::vector<double>(costs, costs + J), tabs, *sys);
    rs::plan::emit(p, out, gpu_cost, sys->num_gpus, summary);
  });
}

int rs_plan_solve(uint32_t J, const rs_plan_table* tables, const rs_system_spec* sys, uint32_t step_count,
                  int use_pooling, int use_coverage, double time_limit_seconds, uint32_t threads,
                  rs_plan_entry* out, double* gpu_cost, rs_plan_summary* summary) {
  return plan_guard([&] {
    if (!sys) rs::plan::invalid("rs_plan_solve: NULL argument");
    if (J == 0) rs::plan::invalid("solve: no tables");
    auto tabs = rs::plan::tables_of(J, tables);
    rs::plan::Abl abl;
    abl.pooling = use_pooling != 0;
    abl.coverage = use_coverage != 0;
    unsigned th = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
    auto p = rs::plan::solve(tabs, *sys, step_count, abl, time_limit_seconds, th);
    rs::plan::emit(p, out, gpu_cost, sys->num_gpus, summary);
  });
}

}  // extern "C"
