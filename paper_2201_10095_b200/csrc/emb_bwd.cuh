// K5 — deterministic sorted-segment backward + optimizer (included by emb.cu).
//
// Input: every lookup of the batch as (key = key_base[t] + storage slot,
// value = sample b), stably radix-sorted by key (scan_sort.cuh).  Table t's
// lookups stay at sorted positions [tpos[t], tpos[t+1]) (the CSR range), and
// every (table, row) is one contiguous SEGMENT of that range.
//
// Reduction tree (restated by oracle.c or_emb_backward), anchored at each
// segment's first position s, length L:
//   L <= 32   g = ((0 + g_s) + g_{s+1}) + ...           (position order, fp32)
//   L > 32    pieces of 32 positions from s, each summed as above; groups of
//             64 consecutive pieces summed left to right (first piece as the
//             accumulator); g = the group sums left to right (first as the
//             accumulator).
// Then row-wise SGD or exact row-wise Adagrad (update_row).  No float atomics:
// results are bitwise reproducible and independent of the launch geometry.
//
// Kernels:
//   seg scan (x2)  warp per 32-position window of a table (class-major order):
//                  count the segment heads, then write one descriptor
//                  {start, key, table} per segment (exclusive scan between)
//   seg            "bags" over segments (the forward's structure: G lanes per
//                  segment, UNR grad-row loads in flight, row + state loaded
//                  first); short segments are summed and updated in place,
//                  long ones are appended to the long list
//   lpiece         warp per 32-position piece of a long segment
//   group          warp per (long segment, group of 64 pieces)
//   long           warp per long segment: sum of its groups, update
#pragma once

namespace rs {
namespace emb {

constexpr int kChunk = 32;        // positions per window / piece
constexpr int kGroupPieces = 64;  // pieces per group of a long segment
constexpr int kBwdThreads = 256;
constexpr int kBwdWarps = kBwdThreads / 32;
constexpr uint32_t kNoKey = 0xFFFFFFFFu;

struct BwdArgs {
  const TableDev* tables;
  uint32_t T;
  const uint32_t* tpos;  // T + 1 sorted-position starts
  const uint32_t* keys;
  const uint32_t* vals;
  const float* grad;
  uint64_t stride;
  uint32_t dmax;
  float lr, eps;
  int opt;
};

__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x = __fadd_rn(a.x, b.x);
  a.y = __fadd_rn(a.y, b.y);
  a.z = __fadd_rn(a.z, b.z);
  a.w = __fadd_rn(a.w, b.w);
}

__device__ __forceinline__ uint32_t upper_index(const uint32_t* v, uint32_t n, uint64_t x) {
  // largest i in [0, n) with v[i] <= x (v ascending, v[0] <= x)
  uint32_t lo = 0, hi = n;
  while (lo + 1 < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (v[mid] <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Optimizer step for one row held by the G lanes of a group (vec = lg+vv*G).
// Arithmetic order matches or_emb_backward: per-lane sum of squares in vec
// order, xor butterfly over the G lanes (= lanes_for(dim) when G is; extra
// lanes hold +0.0f, which leaves q >= 0 unchanged).
template <int G, int VPL, class E>
__device__ __forceinline__ void update_row(const BwdArgs& a, const TableDev& td, int32_t e,
                                           const float4 (&g)[VPL], const float4 (&w)[VPL],
                                           float m_old, unsigned gmask, int lg) {
  const uint32_t V = td.dim >> 2;
  float mult = a.lr;
  if (a.opt == RS_OPT_ROWWISE_ADAGRAD) {
    float q = 0.f;
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) {
      if (uint32_t(lg + vv * G) < V) {
        q = __fadd_rn(q, __fmul_rn(g[vv].x, g[vv].x));
        q = __fadd_rn(q, __fmul_rn(g[vv].y, g[vv].y));
        q = __fadd_rn(q, __fmul_rn(g[vv].z, g[vv].z));
        q = __fadd_rn(q, __fmul_rn(g[vv].w, g[vv].w));
      }
    }
#pragma unroll
    for (int o = G >> 1; o >= 1; o >>= 1) q = __fadd_rn(q, __shfl_xor_sync(gmask, q, o));
    const float m = __fadd_rn(m_old, __fdiv_rn(q, float(td.dim)));
    if (lg == 0) *mom_ptr(td, e) = m;
    mult = __fdiv_rn(a.lr, __fadd_rn(__fsqrt_rn(m), a.eps));
  }
  char* wp = row_ptr(td, e);
#pragma unroll
  for (int vv = 0; vv < VPL; ++vv) {
    const uint32_t vec = lg + vv * G;
    if (vec < V) {
      float4 x = w[vv];
      x.x = __fsub_rn(x.x, __fmul_rn(mult, g[vv].x));
      x.y = __fsub_rn(x.y, __fmul_rn(mult, g[vv].y));
      x.z = __fsub_rn(x.z, __fmul_rn(mult, g[vv].z));
      x.w = __fsub_rn(x.w, __fmul_rn(mult, g[vv].w));
      Elem<E>::store(wp, vec, x);
    }
  }
}

// update_row with the row and state pointers already at hand (the
// short-segment kernel computes them once, before the gradient loads).
template <int G, int VPL, class E>
__device__ __forceinline__ void update_row_at(const BwdArgs& a, uint32_t dim, char* wp, float* mp,
                                              const float4 (&g)[VPL], const float4 (&w)[VPL], float m_old,
                                              unsigned gmask, int lg) {
  const uint32_t V = dim >> 2;
  float mult = a.lr;
  if (a.opt == RS_OPT_ROWWISE_ADAGRAD) {
    float q = 0.f;
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) {
      if (uint32_t(lg + vv * G) < V) {
        q = __fadd_rn(q, __fmul_rn(g[vv].x, g[vv].x));
        q = __fadd_rn(q, __fmul_rn(g[vv].y, g[vv].y));
        q = __fadd_rn(q, __fmul_rn(g[vv].z, g[vv].z));
        q = __fadd_rn(q, __fmul_rn(g[vv].w, g[vv].w));
      }
    }
#pragma unroll
    for (int o = G >> 1; o >= 1; o >>= 1) q = __fadd_rn(q, __shfl_xor_sync(gmask, q, o));
    const float m = __fadd_rn(m_old, __fdiv_rn(q, float(dim)));
    if (lg == 0) *mp = m;
    mult = __fdiv_rn(a.lr, __fadd_rn(__fsqrt_rn(m), a.eps));
  }
#pragma unroll
  for (int vv = 0; vv < VPL; ++vv) {
    const uint32_t vec = lg + vv * G;
    if (vec < V) {
      float4 x = w[vv];
      x.x = __fsub_rn(x.x, __fmul_rn(mult, g[vv].x));
      x.y = __fsub_rn(x.y, __fmul_rn(mult, g[vv].y));
      x.z = __fsub_rn(x.z, __fmul_rn(mult, g[vv].z));
      x.w = __fsub_rn(x.w, __fmul_rn(mult, g[vv].w));
      Elem<E>::store(wp, vec, x);
    }
  }
}

template <int G, int VPL>
__device__ __forceinline__ void store_vec(float* base, uint32_t V, int lg, const float4 (&g)[VPL]) {
  float4* p = reinterpret_cast<float4*>(base);
#pragma unroll
  for (int vv = 0; vv < VPL; ++vv)
    if (uint32_t(lg + vv * G) < V) p[lg + vv * G] = g[vv];
}

template <int G, int VPL>
__device__ __forceinline__ void load_vec(const float* base, uint32_t V, int lg, float4 (&g)[VPL]) {
  const float4* p = reinterpret_cast<const float4*>(base);
#pragma unroll
  for (int vv = 0; vv < VPL; ++vv) {
    const uint32_t vec = lg + vv * G;
    g[vv] = vec < V ? p[vec] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Window work index -> (table, window in table), tables in class-major order.
struct WorkMap {
  const uint32_t* wstart;  // [nt + 1] first work index of each table
  const uint32_t* wtab;    // [nt] table index
  uint32_t nt;
};

// ---------------------------------------------------------------- plan
// Block-wide exclusive scan of one value per thread (blockDim.x = 1024).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sm, uint32_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sm[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t x = lane < int(blockDim.x >> 5) ? sm[lane] : 0u;
    uint32_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    sm[lane] = xi - x;
    if (lane == 31) sm[32] = xi;
  }
  __syncthreads();
  const uint32_t r = sm[wid] + inc - v;
  total = sm[32];
  __syncthreads();
  return r;
}

struct BwdPlan {
  const uint32_t* off;    // the batch's table-major CSR offsets [T*B + 1]
  uint64_t B;
  uint32_t T;
  const uint32_t* order;  // [T] tables in class-major order
  const uint32_t* cpos;   // [ncls + 1] class boundaries in `order`
  uint32_t ncls;
  uint64_t max_lookups;
  uint32_t* tpos;         // [T + 1] sorted-position start of each table
  uint32_t* wstart;       // [T + 1] first window of order[i]
  uint32_t* wtab;         // [T]
  uint32_t* cw;           // [ncls + 1] first window of each class
  uint32_t* tiles;        // sort tiles: pos | cidx | cstride, each `tcap` words
  uint32_t tcap;
  uint32_t* nt;           // sort tile count
  unsigned* err;          // forward bits 1, 2; here 4 (off[0] != 0), 8 (> max_lookups), 16 (decreasing)
};

// One CTA of 1024 threads: everything the backward used to read back to the
// host — validation, the class-major window work map and the segmented sort's
// tile map — computed where the offsets are.  On any error (the forward's
// included) the plan is empty, so every later kernel of the backward does
// nothing and the host raises after the fact.
__global__ void __launch_bounds__(1024) bwd_plan_kernel(BwdPlan p) {
  __shared__ uint32_t sm[33];
  __shared__ unsigned s_err;
  const uint32_t T = p.T;
  if (threadIdx.x == 0) s_err = 0;
  __syncthreads();
  for (uint32_t t = threadIdx.x; t <= T; t += blockDim.x) p.tpos[t] = p.off[uint64_t(t) * p.B];
  __syncthreads();
  unsigned bad = 0;
  for (uint32_t t = threadIdx.x; t < T; t += blockDim.x)
    if (p.tpos[t + 1] < p.tpos[t]) bad |= 16u;
  if (threadIdx.x == 0) {
    if (p.tpos[0] != 0) bad |= 4u;
    if (p.tpos[T] > p.max_lookups) bad |= 8u;
  }
  if (bad) atomicOr(&s_err, bad);
  __syncthreads();
  if (s_err) {
    if (threadIdx.x == 0) atomicOr(p.err, s_err);
  }
  __syncthreads();
  const bool empty = *reinterpret_cast<volatile unsigned*>(p.err) != 0;
  __syncthreads();
  // windows of 32 sorted positions per table, class-major
  uint32_t carry = 0;
  for (uint32_t i0 = 0; i0 < T; i0 += blockDim.x) {
    const uint32_t i = i0 + threadIdx.x;
    uint32_t nw = 0, t = 0;
    if (i < T) {
      t = p.order[i];
      nw = empty ? 0u : (p.tpos[t + 1] - p.tpos[t] + kChunk - 1) / kChunk;
    }
    uint32_t tot;
    const uint32_t x = block_excl_scan(nw, sm, tot);
    if (i < T) {
      p.wstart[i] = carry + x;
      p.wtab[i] = t;
    }
    carry += tot;
  }
  if (threadIdx.x == 0) p.wstart[T] = carry;
  __syncthreads();
  for (uint32_t c = threadIdx.x; c <= p.ncls; c += blockDim.x) p.cw[c] = p.wstart[p.cpos[c]];
  // sort tiles (table order): ceil(L_t / kSortTile) per table
  uint32_t tb = 0;
  for (uint32_t t0 = 0; t0 < T; t0 += blockDim.x) {
    const uint32_t t = t0 + threadIdx.x;
    uint32_t ntt = 0;
    if (t < T && !empty) ntt = (p.tpos[t + 1] - p.tpos[t] + kSortTile - 1) / kSortTile;
    uint32_t tot;
    const uint32_t x = block_excl_scan(ntt, sm, tot);
    // the warp writes its 32 tables' tiles one table at a time, lanes over tiles
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < 32; ++i) {
      const uint32_t ti = __shfl_sync(0xffffffffu, t, i);
      const uint32_t ni = __shfl_sync(0xffffffffu, ntt, i);
      const uint32_t bi = tb + __shfl_sync(0xffffffffu, x, i);
      if (ni == 0) continue;
      const uint32_t start = p.tpos[ti];
      for (uint32_t j = lane; j < ni; j += 32) {
        p.tiles[bi + j] = start + j * kSortTile;
        p.tiles[p.tcap + bi + j] = uint32_t(kRadix) * bi + j;
        p.tiles[2 * p.tcap + bi + j] = ni;
      }
    }
    tb += tot;
  }
  if (threadIdx.x == 0) {
    p.tiles[tb] = empty ? 0u : p.tpos[T];
    *p.nt = tb;
  }
}

// After a stand-alone keygen: an index error it found empties the plan.
__global__ void bwd_plan_gate_kernel(BwdPlan p) {
  if (*reinterpret_cast<volatile unsigned*>(p.err) == 0) return;
  for (uint32_t c = threadIdx.x; c <= p.ncls; c += blockDim.x) p.cw[c] = 0;
  if (threadIdx.x == 0) {
    p.wstart[p.T] = 0;
    p.tiles[0] = 0;
    *p.nt = 0;
  }
}

// ---------------------------------------------------------------- segment list
// WRITE = false: counts[wi] = segment heads in window wi.  WRITE = true: one
// descriptor {start, key, table, end} per head at sbase[wi] + rank (sbase =
// exclusive scan of counts), so each class's segments are contiguous and in
// position order.
template <bool WRITE>
__global__ void __launch_bounds__(256) bwd_seg_scan_kernel(BwdArgs a, WorkMap m, uint32_t* __restrict__ counts,
                                                          const uint32_t* __restrict__ sbase,
                                                          uint4* __restrict__ segs) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwork = m.wstart[m.nt];
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  // each warp walks a contiguous run of windows: one table search per run,
  // then the table index only moves forward (and the keys it reads are
  // consecutive)
  const uint64_t per = (nwork + nwarps - 1) / nwarps;
  const uint64_t w0 = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * per;
  const uint64_t w1 = min(nwork, w0 + per);
  uint32_t i = w0 < w1 ? upper_index(m.wstart, m.nt, w0) : 0u;
  for (uint64_t wi = w0; wi < w1; ++wi) {
    while (m.wstart[i + 1] <= wi) ++i;  // (tables without windows are skipped)
    const uint32_t t = m.wtab[i];
    const uint32_t k = uint32_t(wi - m.wstart[i]);
    const uint32_t tb = a.tpos[t], te = a.tpos[t + 1];
    const uint32_t p0 = tb + k * kChunk;
    const uint32_t n = min(uint32_t(kChunk), te - p0);
    const bool v = uint32_t(lane) < n;
    const uint32_t key = v ? a.keys[p0 + lane] : kNoKey;
    uint32_t kp = __shfl_up_sync(0xffffffffu, key, 1);
    if (lane == 0) kp = p0 > tb ? a.keys[p0 - 1] : kNoKey;
    const bool head = v && key != kp;
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    if (!WRITE) {
      if (lane == 0) counts[wi] = __popc(heads);
      continue;
    }
    // .w = the segment's end: the next head in this window, the table's end
    // when this is its last window, else written by the next window's first
    // head — or by the table's last window when no head follows (descriptor
    // sbase[wi] - 1 is then this one: windows of a table are consecutive work
    // items and a table's first position is always a head).
    if (heads == 0) {
      if (lane == 0 && p0 + uint32_t(kChunk) >= te) reinterpret_cast<uint32_t*>(segs + sbase[wi] - 1)[3] = te;
      continue;
    }
    if (!head) continue;
    const uint32_t idx = sbase[wi] + __popc(heads & lanemask_lt());
    uint4* sd = segs + idx;
    const unsigned later = heads & ~(lanemask_lt() | (1u << lane));
    *reinterpret_cast<uint2*>(sd) = make_uint2(p0 + lane, key);
    if (later) {
      reinterpret_cast<uint32_t*>(sd)[3] = p0 + uint32_t(__ffs(later) - 1);
    } else if (p0 + uint32_t(kChunk) >= te) {
      reinterpret_cast<uint32_t*>(sd)[3] = te;
    }
    reinterpret_cast<uint32_t*>(sd)[2] = t;
    if (k > 0 && (heads & lanemask_lt()) == 0) reinterpret_cast<uint32_t*>(segs + idx - 1)[3] = p0 + lane;
  }
}

// ---------------------------------------------------------------- short segments
// Segments [sbase[w_lo], sbase[w_hi]) of one lane class ({start, key, table,
// end} descriptors from the scan).  Segments
// of <= 32 positions are summed in position order and their row updated;
// longer ones go to the long list (a slot each, with their group count).
template <int G, int VPL, int UNR, int MINB, class E>
__global__ void __launch_bounds__(kBwdThreads, MINB)
bwd_seg_kernel(BwdArgs a, const uint4* __restrict__ segs, const uint32_t* __restrict__ sbase,
               const uint32_t* __restrict__ cw, uint32_t ci, uint4* __restrict__ longs,
               uint32_t* __restrict__ long_np, uint32_t* __restrict__ long_ng, unsigned* __restrict__ n_long) {
  const uint32_t w_lo = cw[ci], w_hi = cw[ci + 1];  // the class's windows (bwd_plan_kernel)
  constexpr int BPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, lg = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const uint64_t s_lo = sbase[w_lo], s_hi = sbase[w_hi];
  const uint32_t npos = a.tpos[a.T];
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const bool ada = a.opt == RS_OPT_ROWWISE_ADAGRAD;
  const uint4 kNone = make_uint4(0u, 0u, kNoKey, 0u);
  // Software pipeline over the grid-stride iterations: the next iteration's
  // descriptor is loaded at the top of this one and its first G sample ids
  // before this segment's update, so an iteration's dependent chain is
  // grad rows -> update (the row and its state are in flight from the top).
  // The table's fields are re-read per segment (L1 hits) instead of being
  // held live across iterations.
  uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  uint4 d = kNone;
  uint32_t smp0 = 0;
  {
    const uint64_t si = s_lo + w * BPW + grp;
    if (si < s_hi) {
      d = segs[si];
      smp0 = a.vals[min(d.x + uint32_t(lg), npos - 1)];
    }
  }
  for (; s_lo + w * BPW < s_hi; w += nwarps) {
    const bool valid = d.z != kNoKey;
    uint4 d2 = kNone;
    {
      const uint64_t si = s_lo + (w + nwarps) * BPW + grp;
      if (si < s_hi) d2 = segs[si];
    }
    const uint32_t len = valid ? d.w - d.x : 0u;
    if (len > uint32_t(kChunk)) {
      if (lg == 0) {
        // a slot, and contiguous ranges of pieces and groups (the reduction
        // tree inside a segment is fixed, so where its range lands does not
        // change any result)
        const uint32_t np = (len + kChunk - 1) / kChunk;
        const unsigned slot = atomicAdd(n_long, 1u);
        longs[slot] = make_uint4(d.x, len, d.y, d.z);
        long_np[slot] = atomicAdd(n_long + 1, np);                                  // first piece
        long_ng[slot] = atomicAdd(n_long + 2, (np + kGroupPieces - 1) / kGroupPieces);  // first group
      }
      smp0 = d2.z != kNoKey ? a.vals[min(d2.x + uint32_t(lg), npos - 1)] : 0u;
      d = d2;
      continue;
    }
    const TableDev& td = a.tables[valid ? d.z : 0u];
    const uint32_t V = td.dim >> 2;
    // the row and its state first: the slot key addresses them directly
    float4 w4[VPL];
    float m_old = 0.f;
    char* wp = nullptr;
    float* mp = nullptr;
    // the unbacked sentinel (key nkeys) has no row: summed like any
    // segment (keeps the warp's shuffles converged), never applied
    const bool upd = valid && d.y < td.nkeys;
    if (upd) {
      // row and state pointers once (fast-tier keys are the row offset)
      if (d.y < td.hbm_rows) {
        wp = td.fast + uint64_t(d.y) * td.rbytes;
        mp = td.mom_fast + d.y;
      } else {
        const int32_t e = entry_of_key(td, d.y);
        wp = row_ptr(td, e);
        mp = mom_ptr(td, e);
      }
#pragma unroll
      for (int vv = 0; vv < VPL; ++vv) {
        const uint32_t vec = lg + vv * G;
        w4[vv] = vec < V ? Elem<E>::load(wp, vec) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (ada) m_old = *mp;
    }
    const float* gcol = a.grad + td.col;
    float4 acc[VPL];
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) acc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (len == 1) {  // most short segments: one gradient row, no unrolled block
      const uint32_t bu = __shfl_sync(gmask, smp0, 0, G);
      const float4* gr = reinterpret_cast<const float4*>(gcol + uint64_t(bu) * a.stride);
#pragma unroll
      for (int vv = 0; vv < VPL; ++vv) {
        const uint32_t vec = lg + vv * G;
        if (vec < V) add4(acc[vv], ld_nc_f4(gr + vec));
      }
    } else
    for (uint32_t base = 0; base < len; base += G) {
      const uint32_t nn = min(uint32_t(G), len - base);
      const uint32_t smp = base == 0 ? smp0 : (uint32_t(lg) < nn ? a.vals[d.x + base + lg] : 0u);
      for (uint32_t j = 0; j < nn; j += UNR) {
        float4 g[UNR][VPL];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint32_t bu = __shfl_sync(gmask, smp, int(j) + u, G);
          const float4* gr = reinterpret_cast<const float4*>(gcol + uint64_t(bu) * a.stride);
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) {
            const uint32_t vec = lg + vv * G;
            g[u][vv] = (j + u < nn && vec < V) ? ld_nc_f4(gr + vec) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          if (j + u < nn) {
#pragma unroll
            for (int vv = 0; vv < VPL; ++vv) add4(acc[vv], g[u][vv]);
          }
      }
    }
    smp0 = d2.z != kNoKey ? a.vals[min(d2.x + uint32_t(lg), npos - 1)] : 0u;
    if (upd) update_row_at<G, VPL, E>(a, td.dim, wp, mp, acc, w4, m_old, gmask, lg);
    d = d2;
  }
}

// ---------------------------------------------------------------- long segments
// Each long slot owns a contiguous range of pieces (first at pfirst[slot])
// and of groups (gfirst[slot]), reserved with atomics by the short-segment
// kernel; n_long = {slots, pieces, groups}.
//
// Warp per long segment: one {start, count, table} descriptor per 32-position
// piece at pdesc[pbase[li] + k], so the piece kernel needs no search.
__global__ void __launch_bounds__(kBwdThreads) bwd_piece_desc_kernel(const uint4* __restrict__ longs,
                                                                    const unsigned* __restrict__ n_long,
                                                                    const uint32_t* __restrict__ pfirst,
                                                                    const uint32_t* __restrict__ gfirst,
                                                                    uint4* __restrict__ pdesc,
                                                                    uint2* __restrict__ gdesc) {
  const int lane = threadIdx.x & 31;
  const uint32_t nl = *n_long;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t li = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; li < nl; li += nwarps) {
    const uint4 L = longs[li];  // {start, len, key, table}
    const uint32_t base = pfirst[li], np = (L.y + kChunk - 1) / kChunk, end = L.x + L.y;
    for (uint32_t k = lane; k < np; k += 32) {
      const uint32_t pb = L.x + k * kChunk;
      pdesc[base + k] = make_uint4(pb, min(uint32_t(kChunk), end - pb), L.w, 0u);
    }
    const uint32_t gb = gfirst[li], ng = (np + kGroupPieces - 1) / kGroupPieces;
    for (uint32_t q = lane; q < ng; q += 32) gdesc[gb + q] = make_uint2(uint32_t(li), q);
  }
}

// Warp per piece (32 positions) of a long segment: summed in position order
// from +0.0f (UNR grad rows in flight), stored to ppart[piece].  Pipelined
// like bwd_seg_kernel: the next piece's descriptor and sample ids are in
// flight while this piece's grad rows are summed.
template <int G, int VPL>
__global__ void __launch_bounds__(kBwdThreads, 3) bwd_lpiece_kernel(BwdArgs a, const uint4* __restrict__ pdesc,
                                                                const unsigned* __restrict__ n_long,
                                                                float* __restrict__ ppart) {
  // G-lane groups (G = 16: two pieces per warp; a dim-128 row is 2 float4
  // per lane, a dim-64 row 1) — the sums are elementwise, so the lane layout
  // does not change any result
  constexpr int BPW = 32 / G;
  constexpr int UNR = 4;  // 4 rows in flight at 3 CTAs/SM beat 8 at 2 (A/B: bwd -0.1-0.2 ms)
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, lg = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const uint32_t nl = n_long[0];
  if (nl == 0) return;
  const uint32_t npieces = n_long[1];
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  uint4 P = make_uint4(0u, 0u, 0u, 0u);
  uint32_t s0 = 0, s1 = 0;  // the piece's sample ids (positions lg, lg + G)
  if (w * BPW + grp < npieces) {
    P = pdesc[w * BPW + grp];
    s0 = uint32_t(lg) < P.y ? a.vals[P.x + lg] : 0u;
    if (G < kChunk) s1 = uint32_t(lg) + G < P.y ? a.vals[P.x + G + lg] : 0u;
  }
  for (; w * BPW < npieces; w += nwarps) {
    const uint64_t pi = w * BPW + grp;
    const bool valid = pi < npieces;
    const uint64_t pn = pi + nwarps * BPW;
    const uint4 Pn = pn < npieces ? pdesc[pn] : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t np = valid ? P.y : 0u;
    const TableDev& td = a.tables[P.z];
    const uint32_t V = td.dim >> 2;
    const float* gcol = a.grad + td.col;
    float4 pc[VPL];
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) pc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int half = 0; half < kChunk / G; ++half) {
      const uint32_t base = uint32_t(half) * G;
      if (base >= np) break;
      const uint32_t nn = min(uint32_t(G), np - base);
      const uint32_t smp = half == 0 ? s0 : s1;
      for (uint32_t j = 0; j < nn; j += UNR) {
        float4 g[UNR][VPL];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint32_t bu = __shfl_sync(gmask, smp, int(j) + u, G);
          const float4* gr = reinterpret_cast<const float4*>(gcol + uint64_t(bu) * a.stride);
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) {
            const uint32_t vec = lg + vv * G;
            g[u][vv] = (j + u < nn && vec < V) ? ld_nc_f4(gr + vec) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          if (j + u < nn) {
#pragma unroll
            for (int vv = 0; vv < VPL; ++vv) add4(pc[vv], g[u][vv]);
          }
      }
    }
    s0 = uint32_t(lg) < Pn.y ? a.vals[Pn.x + lg] : 0u;
    if (G < kChunk) s1 = uint32_t(lg) + G < Pn.y ? a.vals[Pn.x + G + lg] : 0u;
    if (valid) store_vec<G, VPL>(ppart + uint64_t(pi) * a.dmax, V, lg, pc);
    P = Pn;
  }
}

// Warp per (long segment, group of 64 pieces): the group's piece sums left
// to right (first as the accumulator), loads batched 8 deep.
template <int VPL>
__global__ void __launch_bounds__(kBwdThreads) bwd_group_kernel(BwdArgs a, const uint4* __restrict__ longs,
                                                               const unsigned* __restrict__ n_long,
                                                               const uint32_t* __restrict__ pfirst,
                                                               const uint2* __restrict__ gdesc,
                                                               const float* __restrict__ ppart,
                                                               float* __restrict__ gpart) {
  const int lane = threadIdx.x & 31;
  const uint32_t ngroups = n_long[2];
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t gi = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; gi < ngroups; gi += nwarps) {
    const uint2 gd = gdesc[gi];  // {long slot, group within it}
    const uint4 L = longs[gd.x];
    const uint32_t V = a.tables[L.w].dim >> 2;
    const uint32_t np = (L.y + kChunk - 1) / kChunk;
    const uint32_t p0 = pfirst[gd.x] + gd.y * kGroupPieces;
    const uint32_t p1 = min(pfirst[gd.x] + np, p0 + kGroupPieces);
    float4 acc[VPL];
    load_vec<32, VPL>(ppart + uint64_t(p0) * a.dmax, V, lane, acc);
    for (uint32_t p = p0 + 1; p < p1; p += 8) {
      float4 x[8][VPL];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p + u < p1) load_vec<32, VPL>(ppart + uint64_t(p + u) * a.dmax, V, lane, x[u]);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p + u < p1) {
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) add4(acc[vv], x[u][vv]);
        }
    }
    store_vec<32, VPL>(gpart + uint64_t(gi) * a.dmax, V, lane, acc);
  }
}

// Warp per long segment: its group sums left to right (first as the
// accumulator), then the row update.
template <int VPL>
__global__ void __launch_bounds__(kBwdThreads) bwd_long_kernel(BwdArgs a, const uint4* __restrict__ longs,
                                                              const unsigned* __restrict__ n_long,
                                                              const uint32_t* __restrict__ gfirst,
                                                              const float* __restrict__ gpart) {
  const int lane = threadIdx.x & 31;
  const uint32_t nl = *n_long;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t li = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; li < nl; li += nwarps) {
    const uint4 L = longs[li];
    const TableDev& td = a.tables[L.w];
    const uint32_t V = td.dim >> 2;
    if (L.z >= td.nkeys) continue;  // the unbacked sentinel: no row to update
    const int32_t e = entry_of_key(td, L.z);
    float4 w[VPL], acc[VPL], x[VPL];
    {
      const char* wr = row_ptr(td, e);
#pragma unroll
      for (int vv = 0; vv < VPL; ++vv) {
        const uint32_t vec = lane + vv * 32;
        w[vv] = vec < V ? load4(td, wr, vec) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    const float m_old = a.opt == RS_OPT_ROWWISE_ADAGRAD ? *mom_ptr(td, e) : 0.f;
    const uint32_t np = (L.y + kChunk - 1) / kChunk;
    const uint32_t g0 = gfirst[li], g1 = g0 + (np + kGroupPieces - 1) / kGroupPieces;
    load_vec<32, VPL>(gpart + uint64_t(g0) * a.dmax, V, lane, acc);
    for (uint32_t g = g0 + 1; g < g1; ++g) {
      load_vec<32, VPL>(gpart + uint64_t(g) * a.dmax, V, lane, x);
#pragma unroll
      for (int vv = 0; vv < VPL; ++vv) add4(acc[vv], x[vv]);
    }
    if (td.ebytes == 2) update_row<32, VPL, __half>(a, td, e, acc, w, m_old, 0xffffffffu, lane);
    else update_row<32, VPL, float>(a, td, e, acc, w, m_old, 0xffffffffu, lane);
  }
}

}  // namespace emb
}  // namespace rs
