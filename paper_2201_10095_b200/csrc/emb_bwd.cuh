// K5 — deterministic sorted-segment backward + optimizer (included by emb.cu).
//
// Input: every lookup of the batch as (key = key_base[t] + row, value =
// sample b), stably radix-sorted by key (scan_sort.cuh).  Sorting keeps the
// tables in order, so table t's lookups stay at sorted positions
// [tpos[t], tpos[t+1]) = the CSR range [offsets[t*B], offsets[(t+1)*B]), and
// each (table, row) is one contiguous segment in lookup order.
//
// Fixed reduction tree (restated by oracle.c or_emb_backward):
//   level 1  each table's range is cut into 32-position chunks starting at
//            tpos[t]; chunks are numbered globally (cbase[t] + k).  A G-lane
//            group (G = lanes for dim/4 float4s) sums each piece (segment ∩
//            chunk) in order from +0.0f with a segmented running sum;
//   level 2  superchunks of 64 consecutive global chunks: a warp sums, left to
//            right, the chunk-edge pieces of every segment that crosses a
//            chunk edge inside the superchunk;
//   level 3  segments crossing superchunk edges: the superchunk holding the
//            segment's start sums its piece and the following superchunks'
//            pieces left to right.
// A segment is updated (row-wise SGD or exact row-wise Adagrad) by the level
// that completes it.  Level 1 stages the segments completing in a batch of U
// positions in shared memory and updates them together, so the dependent
// remap -> row -> state loads of different rows overlap.  No float atomics;
// results are bitwise reproducible.
#pragma once

namespace rs {
namespace emb {

constexpr int kChunk = 32;
constexpr int kSuper = 64;
constexpr int kBwdThreads = 256;
constexpr int kBwdWarps = kBwdThreads / 32;
constexpr uint32_t kNoKey = 0xFFFFFFFFu;

struct BwdArgs {
  const TableDev* tables;
  uint32_t T;
  const uint32_t* tpos;   // T + 1 sorted-position starts
  const uint32_t* cbase;  // T + 1 global chunk starts
  uint64_t nchunks;       // cbase[T]
  const uint32_t* keys;
  const uint32_t* vals;
  const float* grad;
  uint64_t stride;
  float* part;   // [nchunks][2][dmax]
  float* spart;  // [nsuper][2][dmax]
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

// Position range and neighbour keys of global chunk c (same table only).
struct ChunkInfo {
  uint32_t t, p0, p1;     // table, [p0, p1)
  uint32_t kf, kl;        // first / last key
  uint32_t kprev, knext;  // keys just outside, kNoKey at a table edge
};

__device__ __forceinline__ ChunkInfo chunk_info(const BwdArgs& a, uint64_t c) {
  ChunkInfo ci;
  ci.t = upper_index(a.cbase, a.T, c);
  // skip empty tables sharing the same cbase
  while (ci.t + 1 < a.T && a.cbase[ci.t + 1] <= c) ++ci.t;
  const uint32_t tb = a.tpos[ci.t], te = a.tpos[ci.t + 1];
  ci.p0 = tb + uint32_t(c - a.cbase[ci.t]) * kChunk;
  ci.p1 = min(ci.p0 + uint32_t(kChunk), te);
  ci.kf = a.keys[ci.p0];
  ci.kl = a.keys[ci.p1 - 1];
  ci.kprev = ci.p0 > tb ? a.keys[ci.p0 - 1] : kNoKey;
  ci.knext = ci.p1 < te ? a.keys[ci.p1] : kNoKey;
  return ci;
}

// Optimizer step for one row held by the G lanes of a group (vec = lg+vv*G).
// Arithmetic order matches or_emb_backward: per-lane sum of squares in vec
// order, xor butterfly over the G lanes (= lanes_for(dim) when G is; extra
// lanes hold +0.0f, which leaves q >= 0 unchanged).
template <int G, int VPL>
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
  float4* wp = reinterpret_cast<float4*>(row_ptr(td, e));
#pragma unroll
  for (int vv = 0; vv < VPL; ++vv) {
    const uint32_t vec = lg + vv * G;
    if (vec < V) {
      float4 x = w[vv];
      x.x = __fsub_rn(x.x, __fmul_rn(mult, g[vv].x));
      x.y = __fsub_rn(x.y, __fmul_rn(mult, g[vv].y));
      x.z = __fsub_rn(x.z, __fmul_rn(mult, g[vv].z));
      x.w = __fsub_rn(x.w, __fmul_rn(mult, g[vv].w));
      wp[vec] = x;
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

// Pending complete segments of one full warp (levels 2 and 3).
template <int VPL, int PEND>
struct Pending {
  uint32_t key[PEND];
  uint32_t tab[PEND];
  float4 g[PEND][VPL];
  int n = 0;

  __device__ __forceinline__ void push(uint32_t k, uint32_t t, const float4 (&acc)[VPL]) {
#pragma unroll
    for (int s = 0; s < PEND; ++s)
      if (s == n) {
        key[s] = k;
        tab[s] = t;
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) g[s][vv] = acc[vv];
      }
    ++n;
  }

  __device__ __forceinline__ void flush(const BwdArgs& a) {
    if (n == 0) return;
    const int lane = threadIdx.x & 31;
    int32_t my_e = 0;
#pragma unroll
    for (int s = 0; s < PEND; ++s)
      if (s == lane && s < n) my_e = entry_of_key(a.tables[tab[s]], key[s]);
    float4 w[PEND][VPL];
    float mom[PEND];
#pragma unroll
    for (int s = 0; s < PEND; ++s) {
      const int32_t e = __shfl_sync(0xffffffffu, my_e, s);
      if (s < n) {
        const TableDev& td = a.tables[tab[s]];
        load_vec<32, VPL>(row_ptr(td, e), td.dim >> 2, lane, w[s]);
        mom[s] = a.opt == RS_OPT_ROWWISE_ADAGRAD ? *mom_ptr(td, e) : 0.f;
      }
    }
#pragma unroll
    for (int s = 0; s < PEND; ++s) {
      const int32_t e = __shfl_sync(0xffffffffu, my_e, s);
      if (s < n) update_row<32, VPL>(a, a.tables[tab[s]], e, g[s], w[s], mom[s], 0xffffffffu, lane);
    }
    n = 0;
  }
};

// ---------------------------------------------------------------- level 1
// One G-lane group per chunk of a table of this (G, VPL) class.  Keys and
// samples of the chunk go to shared memory; head/tail masks come from the
// neighbouring keys; rows are gathered U at a time into a segmented running
// sum.  Complete segments are staged and updated together per batch; edge
// pieces go to the level-2 buffer.
template <int G, int VPL, int U, int MINB>
__global__ void __launch_bounds__(kBwdThreads, MINB) bwd_chunk_kernel(BwdArgs a, const uint32_t* cls_tables,
                                                                const uint32_t* cls_cbase, uint32_t ncls) {
  constexpr int GPW = 32 / G;
  constexpr int NGRP = kBwdWarps * GPW;
  // dynamic smem: [NGRP][U][G*VPL] float4 stage, then [NGRP][kChunk+2] keys,
  // then [NGRP][kChunk] samples
  extern __shared__ float4 stage_mem[];
  const int lane = threadIdx.x & 31, lg = lane % G;
  const int gid = (threadIdx.x >> 5) * GPW + lane / G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((lane / G) * G));
  float4* stage = stage_mem + size_t(gid) * U * G * VPL;
  uint32_t* kbase = reinterpret_cast<uint32_t*>(stage_mem + size_t(NGRP) * U * G * VPL);
  uint32_t* sk = kbase + gid * (kChunk + 2) + 1;  // sk[-1] = key before, sk[n] = key after
  uint32_t* sb = kbase + NGRP * (kChunk + 2) + gid * kChunk;
  const uint64_t nwork = cls_cbase[ncls];
  const uint64_t ngroups = uint64_t(gridDim.x) * NGRP;
  for (uint64_t wi = uint64_t(blockIdx.x) * NGRP + gid; wi < nwork; wi += ngroups) {
    const uint32_t j = upper_index(cls_cbase, ncls, wi);
    const uint32_t t = cls_tables[j];
    const uint32_t k = uint32_t(wi - cls_cbase[j]);
    const TableDev td = a.tables[t];
    const uint32_t V = td.dim >> 2;
    const uint32_t tb = a.tpos[t], te = a.tpos[t + 1];
    const uint32_t p0 = tb + k * kChunk;
    const uint32_t n = min(uint32_t(kChunk), te - p0);
    const uint64_t gc = uint64_t(a.cbase[t]) + k;
    __syncwarp(gmask);
    for (uint32_t i = lg; i <= uint32_t(kChunk); i += G) {
      uint32_t kv = kNoKey;
      if (i < n) kv = a.keys[p0 + i];
      else if (i == n && p0 + n < te) kv = a.keys[p0 + n];  // key after (same table)
      sk[i] = kv;
      if (i < uint32_t(kChunk)) sb[i] = i < n ? a.vals[p0 + i] : 0u;
    }
    if (lg == 0) sk[-1] = p0 > tb ? a.keys[p0 - 1] : kNoKey;
    __syncwarp(gmask);
    unsigned heads = 0, tails = 0;
#pragma unroll
    for (int r = 0; r < kChunk / G; ++r) {
      const uint32_t i = lg + r * G;
      const uint32_t kk = sk[i];
      const bool v = i < n;
      const unsigned hb = __ballot_sync(gmask, v && kk != sk[i - 1]);
      const unsigned tb2 = __ballot_sync(gmask, v && kk != sk[i + 1]);
      const unsigned sh = (lane / G) * G;
      heads |= ((hb >> sh) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u))) << (r * G);
      tails |= ((tb2 >> sh) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u))) << (r * G);
    }
    // complete segments end at a tail with a head at or before it (a tail
    // before the first head ends the piece that began in an earlier chunk)
    const int fh = heads ? __ffs(heads) - 1 : 32;
    const unsigned complete = fh >= 32 ? 0u : (tails & ~((1u << fh) - 1u));
    constexpr unsigned UMASK = U >= 32 ? 0xFFFFFFFFu : ((1u << U) - 1u);
    // gathers the grad rows of batch jb (U positions) into v
    auto gather = [&](uint32_t jb, float4 (&v)[U][VPL]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t pos = jb + u;
        const uint32_t bu = sb[pos & (kChunk - 1)];
        const float4* gr = reinterpret_cast<const float4*>(a.grad + uint64_t(bu) * a.stride + td.col);
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) {
          const uint32_t vec = lg + vv * G;
          v[u][vv] = (pos < n && vec < V) ? ld_nc_f4(gr + vec) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    };
    // lane s of the group loads the remap entry of the s-th complete segment of batch jb
    auto remap_of = [&](uint32_t jb) -> int32_t {
      unsigned m = (complete >> jb) & UMASK;
      int32_t e = 0;
#pragma unroll
      for (int s = 0; s < U; ++s) {
        if (m == 0) break;
        const int u = __ffs(m) - 1;
        m &= m - 1;
        if (lg == s) e = entry_of_key(td, sk[jb + u]);
      }
      return e;
    };
    // Software pipeline per batch: the row/state loads of this batch's
    // complete segments and the grad gathers + remap loads of the next batch
    // are all in flight before this batch is summed and updated.
    float4 acc[VPL];
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) acc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 vA[U][VPL], vB[U][VPL];
    gather(0, vA);
    int32_t e_next = remap_of(0);
    for (uint32_t jb = 0; jb < n; jb += U) {
      const unsigned cm = (complete >> jb) & UMASK;
      const int ns = __popc(cm);
      const int32_t e_cur = e_next;
      float4 wv[U][VPL];
      float mom[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int32_t e = __shfl_sync(gmask, e_cur, q % G, G);
        if (q < ns) {
          load_vec<G, VPL>(row_ptr(td, e), V, lg, wv[q]);
          mom[q] = a.opt == RS_OPT_ROWWISE_ADAGRAD ? *mom_ptr(td, e) : 0.f;
        }
      }
      if (jb + U < n) {
        gather(jb + U, vB);
        e_next = remap_of(jb + U);
      }
      int s = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t pos = jb + u;
        if (pos < n) {
          if ((heads >> pos) & 1u) {
#pragma unroll
            for (int vv = 0; vv < VPL; ++vv) acc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) add4(acc[vv], vA[u][vv]);
          if ((tails >> pos) & 1u) {
            if ((cm >> u) & 1u) {
#pragma unroll
              for (int vv = 0; vv < VPL; ++vv) stage[(s * VPL + vv) * G + lg] = acc[vv];
              ++s;
            } else {
              store_vec<G, VPL>(a.part + (gc * 2) * a.dmax, V, lg, acc);  // began before: head edge
            }
          }
        }
      }
      __syncwarp(gmask);
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int32_t e = __shfl_sync(gmask, e_cur, q % G, G);
        if (q < ns) {
          float4 g[VPL];
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) g[vv] = stage[(q * VPL + vv) * G + lg];
          update_row<G, VPL>(a, td, e, g, wv[q], mom[q], gmask, lg);
        }
      }
      __syncwarp(gmask);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) vA[u][vv] = vB[u][vv];
    }
    // the last piece continues into the next chunk: tail edge piece (or the
    // whole chunk is the middle of a segment: head edge piece)
    if (!((tails >> (n - 1)) & 1u)) store_vec<G, VPL>(a.part + (gc * 2 + (heads == 0 ? 0 : 1)) * a.dmax, V, lg, acc);
  }
}

// ---------------------------------------------------------------- level 1, dim <= 128
// Shared-memory staged variant for rows of at most 32 float4 (one per lane of
// a G-lane group).  A group takes a chunk and puts EVERY load of it in flight
// at once with cp.async: the grad rows of all its positions, then (keys are
// storage slots, so no remap load) the rows and Adagrad state of its complete
// segments.  It then sums the pieces from shared memory in position order and
// applies the updates.  Same reduction tree and arithmetic as
// bwd_chunk_kernel; registers stay low, the loads have full memory-level
// parallelism.  Shared memory per group: 2 x 32 x G float4 + 130 words.
constexpr int kGroupWords = 130;  // sk[34] | sb[32] | se[32] | smo[32]

template <int G, int NW>
constexpr size_t chunk_smem_bytes() {
  return size_t(NW) * (32 / G) * (2 * kChunk * G * sizeof(float4) + kGroupWords * 4);
}

template <int G, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
bwd_chunk_smem_kernel(BwdArgs a, const uint32_t* cls_tables, const uint32_t* cls_cbase, uint32_t ncls) {
  constexpr int GPW = 32 / G;
  constexpr int NGRP = NW * GPW;
  extern __shared__ float4 sm5[];
  const int lane = threadIdx.x & 31, lg = lane % G;
  const int gid = (threadIdx.x >> 5) * GPW + lane / G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((lane / G) * G));
  float4* gst = sm5 + size_t(gid) * (2 * kChunk * G);
  float4* wst = gst + kChunk * G;
  uint32_t* ub = reinterpret_cast<uint32_t*>(sm5 + size_t(NGRP) * 2 * kChunk * G) + gid * kGroupWords;
  uint32_t* sk = ub + 1;  // sk[-1] = key before, sk[n] = key after
  uint32_t* sb = ub + kChunk + 2;
  int32_t* se = reinterpret_cast<int32_t*>(ub + 2 * kChunk + 2);
  float* smo = reinterpret_cast<float*>(ub + 3 * kChunk + 2);
  const bool ada = a.opt == RS_OPT_ROWWISE_ADAGRAD;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint64_t nwork = cls_cbase[ncls];
  const uint64_t ngroups = uint64_t(gridDim.x) * NGRP;
  for (uint64_t wi = uint64_t(blockIdx.x) * NGRP + gid; wi < nwork; wi += ngroups) {
    const uint32_t j = upper_index(cls_cbase, ncls, wi);
    const uint32_t t = cls_tables[j];
    const uint32_t k = uint32_t(wi - cls_cbase[j]);
    const TableDev td = a.tables[t];
    const uint32_t V = td.dim >> 2;
    const bool lv = uint32_t(lg) < V;
    const uint32_t tb = a.tpos[t], te = a.tpos[t + 1];
    const uint32_t p0 = tb + k * kChunk;
    const uint32_t n = min(uint32_t(kChunk), te - p0);
    const uint64_t gc = uint64_t(a.cbase[t]) + k;
    __syncwarp(gmask);  // the previous chunk's shared-memory reads are done
    for (uint32_t i = lg; i <= uint32_t(kChunk); i += G) {
      uint32_t kv = kNoKey;
      if (i < n) kv = a.keys[p0 + i];
      else if (i == n && p0 + n < te) kv = a.keys[p0 + n];  // key after (same table)
      sk[i] = kv;
      if (i < uint32_t(kChunk)) sb[i] = i < n ? a.vals[p0 + i] : 0u;
    }
    if (lg == 0) sk[-1] = p0 > tb ? a.keys[p0 - 1] : kNoKey;
    __syncwarp(gmask);
    // 1. every position's grad row (lane lg: float4 lg of the row)
    if (lv) {
      const float* gcol = a.grad + td.col + 4 * lg;
#pragma unroll 8
      for (uint32_t i = 0; i < n; ++i) cp_async16(gst + i * G + lg, gcol + uint64_t(sb[i]) * a.stride);
    }
    cp_async_commit();
    // 2. segment heads / tails inside the chunk
    unsigned heads = 0, tails = 0;
#pragma unroll
    for (int r = 0; r < kChunk / G; ++r) {
      const uint32_t i = lg + r * G;
      const uint32_t kk = sk[i];
      const bool v = i < n;
      const unsigned hb = __ballot_sync(gmask, v && kk != sk[i - 1]);
      const unsigned tb2 = __ballot_sync(gmask, v && kk != sk[i + 1]);
      const unsigned sh = (lane / G) * G;
      heads |= ((hb >> sh) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u))) << (r * G);
      tails |= ((tb2 >> sh) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u))) << (r * G);
    }
    const int fh = heads ? __ffs(heads) - 1 : 32;
    const unsigned complete = fh >= 32 ? 0u : (tails & ~((1u << fh) - 1u));
    const int ns = __popc(complete);
    // 3. rows (+ state) of the complete segments, addressed by their slot keys
    for (uint32_t i = lg; i < n; i += G) {
      if ((complete >> i) & 1u) {
        const int r = __popc(complete & ((1u << i) - 1u));
        const int32_t e = entry_of_key(td, sk[i]);
        se[r] = e;
        if (ada) smo[r] = *mom_ptr(td, e);
      }
    }
    __syncwarp(gmask);
    if (lv)
      for (int r = 0; r < ns; ++r) cp_async16(wst + r * G + lg, row_ptr(td, se[r]) + 4 * lg);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp(gmask);
    // 4. pieces in position order from +0.0f; complete segments update their row
    float4 acc = zero;
    int r = 0;
    for (uint32_t i = 0; i < n; ++i) {
      if ((heads >> i) & 1u) acc = zero;
      if (lv) add4(acc, gst[i * G + lg]);
      if ((tails >> i) & 1u) {
        float4 g1[1] = {acc};
        if ((complete >> i) & 1u) {
          float4 w1[1] = {lv ? wst[r * G + lg] : zero};
          update_row<G, 1>(a, td, se[r], g1, w1, smo[r], gmask, lg);
          ++r;
        } else {
          store_vec<G, 1>(a.part + (gc * 2) * a.dmax, V, lg, g1);  // began before: head edge
        }
      }
    }
    if (!((tails >> (n - 1)) & 1u)) {
      float4 g1[1] = {acc};
      store_vec<G, 1>(a.part + (gc * 2 + (heads == 0 ? 0 : 1)) * a.dmax, V, lg, g1);
    }
  }
}

// ---------------------------------------------------------------- level 1 as bags
// Level 1 restated as an EmbeddingBag over the grad matrix: every PIECE
// (segment ∩ chunk) is a bag of <= 32 positions whose "indices" are the
// samples of its lookups.  A scan pass (warp per chunk, lane per position)
// lists the pieces; the bag pass gathers each piece's grad rows with the
// forward's structure (G lanes per piece, UNR row loads in flight, in-order
// fp32 adds from +0.0f) and either updates the row (the piece is a whole
// segment: row and state loads are issued first, addressed by the slot key)
// or stores the edge piece for level 2.  Same tree as bwd_chunk_kernel.
constexpr uint32_t kPieceComplete = 0, kPieceSlot0 = 1, kPieceSlot1 = 2;

// Chunk work index -> (table, chunk in table), tables in class-major order.
struct WorkMap {
  const uint32_t* wstart;  // [nt + 1] first work index of each table
  const uint32_t* wtab;    // [nt] table index
  uint32_t nt;
};

// WRITE = false: counts[wi] = pieces of chunk wi.  WRITE = true: pieces at
// pbase[wi] (exclusive scan of counts) as {start, global chunk, key, table << 8 | type << 6 | len - 1}.
template <bool WRITE>
__global__ void __launch_bounds__(256) bwd_piece_scan_kernel(BwdArgs a, WorkMap m, uint32_t* __restrict__ counts,
                                                            const uint32_t* __restrict__ pbase,
                                                            uint4* __restrict__ pieces) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwork = m.wstart[m.nt];
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t wi = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; wi < nwork; wi += nwarps) {
    const uint32_t i = upper_index(m.wstart, m.nt, wi);
    const uint32_t t = m.wtab[i];
    const uint32_t k = uint32_t(wi - m.wstart[i]);
    const uint32_t tb = a.tpos[t], te = a.tpos[t + 1];
    const uint32_t p0 = tb + k * kChunk;
    const uint32_t n = min(uint32_t(kChunk), te - p0);
    const bool v = uint32_t(lane) < n;
    const uint32_t key = v ? a.keys[p0 + lane] : kNoKey;
    uint32_t kp = __shfl_up_sync(0xffffffffu, key, 1);
    if (lane == 0) kp = p0 > tb ? a.keys[p0 - 1] : kNoKey;
    uint32_t kn = __shfl_down_sync(0xffffffffu, key, 1);
    if (uint32_t(lane) == n - 1) kn = p0 + n < te ? a.keys[p0 + n] : kNoKey;
    const bool head = v && key != kp;
    const unsigned starts = __ballot_sync(0xffffffffu, v && (lane == 0 || head));
    const unsigned tails = __ballot_sync(0xffffffffu, v && key != kn);
    if (!WRITE) {
      if (lane == 0) counts[wi] = __popc(starts);
      continue;
    }
    if ((starts >> lane) & 1u) {
      const unsigned rest = lane < 31 ? (starts >> (lane + 1)) : 0u;
      const uint32_t e = rest ? uint32_t(lane) + __ffs(rest) : n;  // end (exclusive)
      const uint32_t type = !head ? kPieceSlot0 : (((tails >> (e - 1)) & 1u) ? kPieceComplete : kPieceSlot1);
      const uint32_t r = __popc(starts & lanemask_lt());
      // {first position, global chunk, slot key, table << 8 | type << 6 | (len - 1)}
      pieces[pbase[wi] + r] = make_uint4(p0 + lane, a.cbase[t] + k, key, (t << 8) | (type << 6) | (e - lane - 1));
    }
  }
}

template <int G, int VPL, int UNR, int MINB>
__global__ void __launch_bounds__(kBwdThreads, MINB)
bwd_piece_kernel(BwdArgs a, const uint4* __restrict__ pieces, const uint32_t* __restrict__ pbase,
                 uint32_t w_lo, uint32_t w_hi) {
  constexpr int BPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, lg = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const uint64_t p_lo = pbase[w_lo], p_hi = pbase[w_hi];
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const bool ada = a.opt == RS_OPT_ROWWISE_ADAGRAD;
  uint32_t cur_t = 0xFFFFFFFFu;
  TableDev td{};
  uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  // the next piece's descriptor is loaded while this one runs
  uint4 dn = p_lo + w * BPW + grp < p_hi ? pieces[p_lo + w * BPW + grp] : make_uint4(0u, 0u, 0u, 0xFFFFFFFFu);
  for (; p_lo + w * BPW < p_hi; w += nwarps) {
    const uint64_t pi = p_lo + w * BPW + grp;
    const bool valid = pi < p_hi;
    const uint4 d = dn;
    {
      const uint64_t pn = pi + nwarps * BPW;
      dn = pn < p_hi ? pieces[pn] : make_uint4(0u, 0u, 0u, 0xFFFFFFFFu);
    }
    const uint32_t len = (d.w & 63u) + 1, type = (d.w >> 6) & 3u, tt = d.w >> 8;
    if (valid && tt != cur_t) {
      cur_t = tt;
      td = a.tables[cur_t];
    }
    const uint32_t V = td.dim >> 2;
    const bool upd = valid && type == kPieceComplete;
    // the row and its state first: the slot key addresses them directly
    float4 w4[VPL];
    float m_old = 0.f;
    int32_t e = 0;
    if (upd) {
      e = entry_of_key(td, d.z);
      const float4* wr = reinterpret_cast<const float4*>(row_ptr(td, e));
#pragma unroll
      for (int vv = 0; vv < VPL; ++vv) {
        const uint32_t vec = lg + vv * G;
        w4[vv] = vec < V ? wr[vec] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (ada) m_old = *mom_ptr(td, e);
    }
    float4 acc[VPL];
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) acc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t base = 0; valid && base < len; base += G) {
      const uint32_t nn = min(uint32_t(G), len - base);
      const uint32_t smp = uint32_t(lg) < nn ? a.vals[d.x + base + lg] : 0u;
      for (uint32_t j = 0; j < nn; j += UNR) {
        float4 g[UNR][VPL];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint32_t bu = __shfl_sync(gmask, smp, int(j) + u, G);
          const float4* gr = reinterpret_cast<const float4*>(a.grad + uint64_t(bu) * a.stride + td.col);
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
    if (upd) update_row<G, VPL>(a, td, e, acc, w4, m_old, gmask, lg);
    else if (valid) store_vec<G, VPL>(a.part + (uint64_t(d.y) * 2 + (type == kPieceSlot1)) * a.dmax, V, lg, acc);
  }
}

// ---------------------------------------------------------------- level 2
// Chunk edge items of superchunk s, in order: per chunk [slot0 head piece]
// [slot1 tail piece].  Runs of equal key are summed left to right.
template <int VPL, int PEND>
__global__ void __launch_bounds__(kBwdThreads, 2) bwd_super_kernel(BwdArgs a) {
  const int lane = threadIdx.x & 31;
  const uint64_t nsuper = (a.nchunks + kSuper - 1) / kSuper;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  Pending<VPL, PEND> pend;
  for (uint64_t s = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; s < nsuper; s += nwarps) {
    const uint64_t cb = s * kSuper, ce = min(cb + kSuper, a.nchunks);
    // lane l describes chunks cb + l and cb + 32 + l
    uint32_t kf[2], kl[2], tt[2];
    unsigned h0[2], h1[2];
    uint32_t kprev = kNoKey, knext = kNoKey;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t c = cb + h * 32 + lane;
      kf[h] = kl[h] = tt[h] = 0;
      h0[h] = h1[h] = 0;
      if (c < ce) {
        const ChunkInfo ci = chunk_info(a, c);
        kf[h] = ci.kf;
        kl[h] = ci.kl;
        tt[h] = ci.t;
        const bool b0 = ci.kprev == ci.kf;
        const bool a1 = ci.knext == ci.kl;
        h0[h] = b0;
        h1[h] = a1 && !(b0 && ci.kf == ci.kl);
        if (c == cb) kprev = ci.kprev;
        if (c == ce - 1) knext = ci.knext;
      }
    }
    kprev = __shfl_sync(0xffffffffu, kprev, 0);
    knext = __shfl_sync(0xffffffffu, knext, int((ce - 1 - cb) & 31));
    uint32_t run = kNoKey;
    bool open = false;
    float4 acc[VPL];
    uint32_t V = 0, t = 0;
    auto close = [&]() {
      if (!open) return;
      const bool before = run == kprev;
      const bool after = run == knext;
      if (!before && !after) {
        pend.push(run, t, acc);
        if (pend.n == PEND) pend.flush(a);
      } else {
        store_vec<32, VPL>(a.spart + (s * 2 + (before ? 0 : 1)) * a.dmax, V, lane, acc);
      }
      open = false;
    };
    for (uint64_t c = cb; c < ce; ++c) {
      const int src = int((c - cb) & 31), hh = int((c - cb) >> 5);
      const uint32_t f0 = __shfl_sync(0xffffffffu, hh ? kf[1] : kf[0], src);
      const uint32_t f1 = __shfl_sync(0xffffffffu, hh ? kl[1] : kl[0], src);
      const uint32_t tc = __shfl_sync(0xffffffffu, hh ? tt[1] : tt[0], src);
      const unsigned e0 = __shfl_sync(0xffffffffu, hh ? h0[1] : h0[0], src);
      const unsigned e1 = __shfl_sync(0xffffffffu, hh ? h1[1] : h1[0], src);
#pragma unroll
      for (int slot = 0; slot < 2; ++slot) {
        const bool has = slot == 0 ? e0 : e1;
        if (!has) continue;
        const uint32_t kk = slot == 0 ? f0 : f1;
        float4 x[VPL];
        if (!open || kk != run) {
          close();
          run = kk;
          open = true;
          t = tc;
          V = a.tables[t].dim >> 2;
          load_vec<32, VPL>(a.part + (c * 2 + slot) * a.dmax, V, lane, acc);
        } else {
          load_vec<32, VPL>(a.part + (c * 2 + slot) * a.dmax, V, lane, x);
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) add4(acc[vv], x[vv]);
        }
      }
    }
    close();
  }
  pend.flush(a);
}

// ---------------------------------------------------------------- level 3
template <int VPL, int PEND>
__global__ void __launch_bounds__(kBwdThreads, 2) bwd_final_kernel(BwdArgs a) {
  const int lane = threadIdx.x & 31;
  const uint64_t nsuper = (a.nchunks + kSuper - 1) / kSuper;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  Pending<VPL, PEND> pend;
  for (uint64_t s = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; s < nsuper; s += nwarps) {
    const uint64_t cb = s * kSuper, ce = min(cb + kSuper, a.nchunks);
    const ChunkInfo last = chunk_info(a, ce - 1);
    if (last.knext != last.kl) continue;  // ends inside
    const ChunkInfo first = chunk_info(a, cb);
    const uint32_t kl = last.kl;
    if (first.kprev == kl && first.kf == kl) continue;  // middle piece
    const uint32_t t = last.t;
    const uint32_t V = a.tables[t].dim >> 2;
    float4 acc[VPL], x[VPL];
    load_vec<32, VPL>(a.spart + (s * 2 + 1) * a.dmax, V, lane, acc);
    for (uint64_t s2 = s + 1; s2 < nsuper; ++s2) {
      load_vec<32, VPL>(a.spart + (s2 * 2) * a.dmax, V, lane, x);
#pragma unroll
      for (int vv = 0; vv < VPL; ++vv) add4(acc[vv], x[vv]);
      const ChunkInfo l2 = chunk_info(a, min((s2 + 1) * kSuper, a.nchunks) - 1);
      if (l2.knext != kl) break;
    }
    pend.push(kl, t, acc);
    if (pend.n == PEND) pend.flush(a);
  }
  pend.flush(a);
}

}  // namespace emb
}  // namespace rs
