// K5 — deterministic sorted-segment backward + optimizer (included by emb.cu).
//
// Input: every lookup of the batch as (key = key_base[t] + row, value =
// sample b), stably radix-sorted by key (scan_sort.cuh), so each (table, row)
// is one contiguous segment of the sorted list in lookup order.
//
// Fixed reduction tree (restated by oracle.c or_emb_backward):
//   level 1  the list is cut into 64-position chunks; a warp per chunk sums
//            each piece (segment ∩ chunk) over its positions in order from
//            +0.0f, gathering grad_out rows 8 at a time;
//   level 2  64-chunk superchunks: a warp sums, left to right, the chunk-edge
//            pieces of every segment that crosses a chunk edge inside it;
//   level 3  segments crossing superchunk edges: the superchunk holding the
//            segment's start sums its piece and the following superchunks'
//            pieces left to right.
// A segment is updated (row-wise SGD or exact row-wise Adagrad) by the level
// that completes it.  Updates are batched PEND at a time per warp so the
// dependent remap -> row -> state loads of different rows overlap.  No float
// atomics; results are bitwise reproducible.
#pragma once

namespace rs {
namespace emb {

constexpr int kChunk = 64;
constexpr int kSuper = 64;
constexpr uint64_t kSpan = uint64_t(kChunk) * kSuper;
constexpr uint32_t kSmemTables = 2048;
constexpr int kBwdThreads = 256;
constexpr int kBwdWarps = kBwdThreads / 32;

struct BwdArgs {
  const TableDev* tables;
  const uint32_t* key_base;  // T + 1 (last = total keys)
  const uint32_t* col;       // T
  const uint32_t* dim;       // T
  uint32_t T;
  const uint32_t* keys;
  const uint32_t* vals;
  uint64_t L;
  const float* grad;
  uint64_t stride;
  float* part;   // [nchunks][2][dmax]
  float* spart;  // [nsuper][2][dmax]
  uint32_t dmax;
  float lr, eps;
  int opt;
};

struct TabView {
  const uint32_t* kb;
  const uint32_t* col;
  const uint32_t* dim;
  uint32_t T;
  __device__ __forceinline__ uint32_t find(uint32_t key) const {  // largest t: kb[t] <= key
    uint32_t lo = 0, hi = T;
    while (lo + 1 < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (kb[mid] <= key) lo = mid;
      else hi = mid;
    }
    return lo;
  }
};

struct TabSmem {
  uint32_t kb[kSmemTables + 1];
  uint32_t col[kSmemTables];
  uint32_t dim[kSmemTables];
};

__device__ __forceinline__ TabView load_tables(const BwdArgs& a, TabSmem& s) {
  if (a.T > kSmemTables) return TabView{a.key_base, a.col, a.dim, a.T};
  for (uint32_t i = threadIdx.x; i <= a.T; i += blockDim.x) {
    s.kb[i] = a.key_base[i];
    if (i < a.T) {
      s.col[i] = a.col[i];
      s.dim[i] = a.dim[i];
    }
  }
  __syncthreads();
  return TabView{s.kb, s.col, s.dim, a.T};
}

__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x = __fadd_rn(a.x, b.x);
  a.y = __fadd_rn(a.y, b.y);
  a.z = __fadd_rn(a.z, b.z);
  a.w = __fadd_rn(a.w, b.w);
}

// Pending complete segments of one warp: key, table and the gradient slice
// (VPL float4 per lane, vec = lane + vv*32).
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

  // Row-wise SGD / exact row-wise Adagrad on every pending row; the loads of
  // all rows are issued before any row is updated.
  __device__ __forceinline__ void flush(const BwdArgs& a) {
    if (n == 0) return;
    const int lane = threadIdx.x & 31;
    int32_t my_e = 0;
#pragma unroll
    for (int s = 0; s < PEND; ++s)
      if (s == lane && s < n) my_e = a.tables[tab[s]].remap[key[s] - a.tables[tab[s]].key_base];
    float4 w[PEND][VPL];
    float mom[PEND];
    float4* wp[PEND];
    float* mp[PEND];
    uint32_t Vs[PEND], Ds[PEND];
#pragma unroll
    for (int s = 0; s < PEND; ++s) {
      const int32_t e = __shfl_sync(0xffffffffu, my_e, s);
      if (s < n) {
        const TableDev& td = a.tables[tab[s]];
        Ds[s] = td.dim;
        Vs[s] = td.dim >> 2;
        wp[s] = reinterpret_cast<float4*>(row_ptr(td, e));
        mp[s] = a.opt == RS_OPT_ROWWISE_ADAGRAD ? mom_ptr(td, e) : nullptr;
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) {
          const uint32_t vec = lane + vv * 32;
          w[s][vv] = vec < Vs[s] ? wp[s][vec] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        mom[s] = mp[s] ? *mp[s] : 0.f;
      }
    }
#pragma unroll
    for (int s = 0; s < PEND; ++s) {
      if (s < n) {
        float mult = a.lr;
        if (a.opt == RS_OPT_ROWWISE_ADAGRAD) {
          float q = 0.f;
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) {
            if (uint32_t(lane + vv * 32) < Vs[s]) {
              q = __fadd_rn(q, __fmul_rn(g[s][vv].x, g[s][vv].x));
              q = __fadd_rn(q, __fmul_rn(g[s][vv].y, g[s][vv].y));
              q = __fadd_rn(q, __fmul_rn(g[s][vv].z, g[s][vv].z));
              q = __fadd_rn(q, __fmul_rn(g[s][vv].w, g[s][vv].w));
            }
          }
          const int Lw = lanes_for(Ds[s]);
          for (int o = Lw >> 1; o >= 1; o >>= 1) q = __fadd_rn(q, __shfl_xor_sync(0xffffffffu, q, o));
          const float m = __fadd_rn(mom[s], __fdiv_rn(q, float(Ds[s])));
          if (lane == 0) *mp[s] = m;
          mult = __fdiv_rn(a.lr, __fadd_rn(__fsqrt_rn(m), a.eps));
        }
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) {
          const uint32_t vec = lane + vv * 32;
          if (vec < Vs[s]) {
            float4 x = w[s][vv];
            x.x = __fsub_rn(x.x, __fmul_rn(mult, g[s][vv].x));
            x.y = __fsub_rn(x.y, __fmul_rn(mult, g[s][vv].y));
            x.z = __fsub_rn(x.z, __fmul_rn(mult, g[s][vv].z));
            x.w = __fsub_rn(x.w, __fmul_rn(mult, g[s][vv].w));
            wp[s][vec] = x;
          }
        }
      }
    }
    n = 0;
  }
};

template <int VPL>
__device__ __forceinline__ void store_vec(float* base, uint32_t V, const float4 (&g)[VPL]) {
  const int lane = threadIdx.x & 31;
  float4* p = reinterpret_cast<float4*>(base);
#pragma unroll
  for (int vv = 0; vv < VPL; ++vv)
    if (uint32_t(lane + vv * 32) < V) p[lane + vv * 32] = g[vv];
}

template <int VPL>
__device__ __forceinline__ void load_vec(const float* base, uint32_t V, float4 (&g)[VPL]) {
  const int lane = threadIdx.x & 31;
  const float4* p = reinterpret_cast<const float4*>(base);
#pragma unroll
  for (int vv = 0; vv < VPL; ++vv) {
    const uint32_t vec = lane + vv * 32;
    g[vv] = vec < V ? p[vec] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// ---------------------------------------------------------------- level 1
template <int VPL, int PEND>
__global__ void __launch_bounds__(kBwdThreads, 2) bwd_chunk_kernel(BwdArgs a) {
  __shared__ TabSmem ts;
  __shared__ uint32_t s_k[kBwdWarps][kChunk], s_v[kBwdWarps][kChunk];
  const TabView tv = load_tables(a, ts);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t nchunks = (a.L + kChunk - 1) / kChunk;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  Pending<VPL, PEND> pend;
  for (uint64_t c = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < nchunks; c += nwarps) {
    const uint64_t c0 = c * kChunk;
    const uint64_t c1 = min(c0 + kChunk, a.L);
    const uint32_t n = uint32_t(c1 - c0);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < kChunk / 32; ++h) {
      const uint64_t i = c0 + h * 32 + lane;
      s_k[w][h * 32 + lane] = i < c1 ? a.keys[i] : 0xFFFFFFFFu;
      s_v[w][h * 32 + lane] = i < c1 ? a.vals[i] : 0u;
    }
    const uint32_t key_before = c0 > 0 ? a.keys[c0 - 1] : 0xFFFFFFFFu;
    const uint32_t key_after = c1 < a.L ? a.keys[c1] : 0xFFFFFFFFu;
    __syncwarp();
    uint32_t cur = s_k[w][0];
    uint32_t t = tv.find(cur);
    uint32_t tend = tv.kb[t + 1];
    uint32_t V = tv.dim[t] >> 2;
    uint32_t tg = t;  // gather-side table cursor (keys ascend)
    float4 acc[VPL];
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) acc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto end_piece = [&](uint32_t pend_pos) {
      const bool before = cur == key_before;
      const bool after = pend_pos == n && cur == key_after;
      if (!before && !after) {
        pend.push(cur, t, acc);
        if (pend.n == PEND) pend.flush(a);
      } else {
        store_vec<VPL>(a.part + (c * 2 + (before ? 0 : 1)) * a.dmax, V, acc);
      }
    };
    for (uint32_t j = 0; j < n; j += 8) {
      float4 v[8][VPL];
      uint32_t ku[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t pos = j + u;
        ku[u] = 0xFFFFFFFFu;
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) v[u][vv] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (pos < n) {
          const uint32_t k = s_k[w][pos];
          const uint32_t b = s_v[w][pos];
          while (k >= tv.kb[tg + 1]) ++tg;
          ku[u] = k;
          const float4* gr = reinterpret_cast<const float4*>(a.grad + uint64_t(b) * a.stride + tv.col[tg]);
          const uint32_t Vu = tv.dim[tg] >> 2;
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) {
            const uint32_t vec = lane + vv * 32;
            if (vec < Vu) v[u][vv] = ld_nc_f4(gr + vec);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t pos = j + u;
        if (pos >= n) break;
        if (ku[u] != cur) {
          end_piece(pos);
          cur = ku[u];
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) acc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (cur >= tend) {
            t = tv.find(cur);
            tend = tv.kb[t + 1];
            V = tv.dim[t] >> 2;
          }
        }
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) add4(acc[vv], v[u][vv]);
      }
    }
    end_piece(n);
  }
  pend.flush(a);
}

// ---------------------------------------------------------------- level 2
// Chunk edge items of superchunk s, in order: per chunk [slot0 head piece]
// [slot1 tail piece].  Runs of equal key are summed left to right.
template <int VPL, int PEND>
__global__ void __launch_bounds__(kBwdThreads, 2) bwd_super_kernel(BwdArgs a) {
  __shared__ TabSmem ts;
  const TabView tv = load_tables(a, ts);
  const int lane = threadIdx.x & 31;
  const uint64_t nchunks = (a.L + kChunk - 1) / kChunk;
  const uint64_t nsuper = (nchunks + kSuper - 1) / kSuper;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  Pending<VPL, PEND> pend;
  for (uint64_t s = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; s < nsuper; s += nwarps) {
    const uint64_t cb = s * kSuper, ce = min(cb + kSuper, nchunks);
    const uint64_t P0 = cb * kChunk, P1 = min(ce * kChunk, a.L);
    const uint32_t kprev = P0 > 0 ? a.keys[P0 - 1] : 0xFFFFFFFFu;
    const uint32_t knext = P1 < a.L ? a.keys[P1] : 0xFFFFFFFFu;
    // per-chunk edge flags: lane l describes chunks cb + l and cb + 32 + l
    uint32_t kf[2], kl[2];
    unsigned h0[2], h1[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t c = cb + h * 32 + lane;
      kf[h] = kl[h] = 0;
      h0[h] = h1[h] = 0;
      if (c < ce) {
        const uint64_t q0 = c * kChunk, q1 = min(q0 + kChunk, a.L);
        kf[h] = a.keys[q0];
        kl[h] = a.keys[q1 - 1];
        const bool b0 = q0 > 0 && a.keys[q0 - 1] == kf[h];
        const bool a1 = q1 < a.L && a.keys[q1] == kl[h];
        h0[h] = b0;
        h1[h] = a1 && !(b0 && kf[h] == kl[h]);
      }
    }
    uint32_t run = 0xFFFFFFFFu;
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
        store_vec<VPL>(a.spart + (s * 2 + (before ? 0 : 1)) * a.dmax, V, acc);
      }
      open = false;
    };
    for (uint64_t c = cb; c < ce; ++c) {
      const int src = int((c - cb) & 31), hh = int((c - cb) >> 5);
      const uint32_t f0 = __shfl_sync(0xffffffffu, hh ? kf[1] : kf[0], src);
      const uint32_t f1 = __shfl_sync(0xffffffffu, hh ? kl[1] : kl[0], src);
      const unsigned e0 = __shfl_sync(0xffffffffu, hh ? h0[1] : h0[0], src);
      const unsigned e1 = __shfl_sync(0xffffffffu, hh ? h1[1] : h1[0], src);
#pragma unroll
      for (int slot = 0; slot < 2; ++slot) {
        const bool has = slot == 0 ? e0 : e1;
        if (!has) continue;
        const uint32_t k = slot == 0 ? f0 : f1;
        float4 x[VPL];
        if (!open || k != run) {
          close();
          run = k;
          open = true;
          t = tv.find(k);
          V = tv.dim[t] >> 2;
          load_vec<VPL>(a.part + (c * 2 + slot) * a.dmax, V, acc);
        } else {
          load_vec<VPL>(a.part + (c * 2 + slot) * a.dmax, V, x);
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
  __shared__ TabSmem ts;
  const TabView tv = load_tables(a, ts);
  const uint64_t nchunks = (a.L + kChunk - 1) / kChunk;
  const uint64_t nsuper = (nchunks + kSuper - 1) / kSuper;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  Pending<VPL, PEND> pend;
  for (uint64_t s = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; s < nsuper; s += nwarps) {
    const uint64_t P0 = s * kSpan, P1 = min(P0 + kSpan, a.L);
    if (P1 >= a.L) continue;
    const uint32_t kl = a.keys[P1 - 1];
    if (a.keys[P1] != kl) continue;                              // ends inside
    if (P0 > 0 && a.keys[P0 - 1] == kl && a.keys[P0] == kl) continue;  // middle piece
    const uint32_t t = tv.find(kl);
    const uint32_t V = tv.dim[t] >> 2;
    float4 acc[VPL], x[VPL];
    load_vec<VPL>(a.spart + (s * 2 + 1) * a.dmax, V, acc);
    for (uint64_t s2 = s + 1; s2 < nsuper; ++s2) {
      load_vec<VPL>(a.spart + (s2 * 2) * a.dmax, V, x);
#pragma unroll
      for (int vv = 0; vv < VPL; ++vv) add4(acc[vv], x[vv]);
      const uint64_t e2 = min((s2 + 1) * kSpan, a.L);
      if (e2 >= a.L || a.keys[e2] != kl) break;
    }
    pend.push(kl, t, acc);
    if (pend.n == PEND) pend.flush(a);
  }
  pend.flush(a);
}

}  // namespace emb
}  // namespace rs
