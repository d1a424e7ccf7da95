// K5 — deterministic sorted-segment backward + optimizer (included by emb.cu).
//
// Input: every lookup of the batch as (key = key_base[t] + row, value =
// sample b), stably radix-sorted by key (scan_sort.cuh), so each (table, row)
// is one contiguous segment of the sorted list in lookup order.
//
// Fixed reduction tree (restated by oracle.c or_emb_backward):
//   level 1  the list is cut into 32-position chunks; a warp per chunk sums
//            each piece (segment ∩ chunk) over its positions in order from
//            +0.0f with a segmented running sum;
//   level 2  64-chunk superchunks: a warp sums, left to right, the chunk-edge
//            pieces of every segment that crosses a chunk edge inside it;
//   level 3  segments crossing superchunk edges: the superchunk holding the
//            segment's start sums its piece and the following superchunks'
//            pieces left to right.
// A segment is updated (row-wise SGD or exact row-wise Adagrad) by the level
// that completes it.  Level 1 stages the segments completing in a batch of
// positions in shared memory and updates them together, so the dependent
// remap -> row -> state loads of different rows overlap.  No float atomics;
// results are bitwise reproducible.
#pragma once

namespace rs {
namespace emb {

constexpr int kChunk = 32;
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

// One row's optimizer step given its full gradient slice g (vec = lane+vv*32)
// and the row's current values w / state m already loaded.  Arithmetic order
// matches or_emb_backward.
template <int VPL>
__device__ __forceinline__ void update_row(const BwdArgs& a, uint32_t dim, const float4 (&g)[VPL],
                                           float4 (&w)[VPL], float m_old, float* mp, float4* wp) {
  const int lane = threadIdx.x & 31;
  const uint32_t V = dim >> 2;
  float mult = a.lr;
  if (a.opt == RS_OPT_ROWWISE_ADAGRAD) {
    float q = 0.f;
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) {
      if (uint32_t(lane + vv * 32) < V) {
        q = __fadd_rn(q, __fmul_rn(g[vv].x, g[vv].x));
        q = __fadd_rn(q, __fmul_rn(g[vv].y, g[vv].y));
        q = __fadd_rn(q, __fmul_rn(g[vv].z, g[vv].z));
        q = __fadd_rn(q, __fmul_rn(g[vv].w, g[vv].w));
      }
    }
    const int Lw = lanes_for(dim);
    for (int o = Lw >> 1; o >= 1; o >>= 1) q = __fadd_rn(q, __shfl_xor_sync(0xffffffffu, q, o));
    const float m = __fadd_rn(m_old, __fdiv_rn(q, float(dim)));
    if (lane == 0) *mp = m;
    mult = __fdiv_rn(a.lr, __fadd_rn(__fsqrt_rn(m), a.eps));
  }
#pragma unroll
  for (int vv = 0; vv < VPL; ++vv) {
    const uint32_t vec = lane + vv * 32;
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

// Pending complete segments of one warp (levels 2 and 3): key, table and the
// gradient slice (VPL float4 per lane, vec = lane + vv*32).
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
      if (s == lane && s < n) my_e = a.tables[tab[s]].remap[key[s] - a.tables[tab[s]].key_base];
    float4 w[PEND][VPL];
    float mom[PEND];
#pragma unroll
    for (int s = 0; s < PEND; ++s) {
      const int32_t e = __shfl_sync(0xffffffffu, my_e, s);
      if (s < n) {
        const TableDev& td = a.tables[tab[s]];
        const float4* wp = reinterpret_cast<const float4*>(row_ptr(td, e));
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) {
          const uint32_t vec = lane + vv * 32;
          w[s][vv] = vec < (td.dim >> 2) ? wp[vec] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        mom[s] = a.opt == RS_OPT_ROWWISE_ADAGRAD ? *mom_ptr(td, e) : 0.f;
      }
    }
#pragma unroll
    for (int s = 0; s < PEND; ++s) {
      const int32_t e = __shfl_sync(0xffffffffu, my_e, s);
      if (s < n) {
        const TableDev& td = a.tables[tab[s]];
        update_row<VPL>(a, td.dim, g[s], w[s], mom[s],
                        a.opt == RS_OPT_ROWWISE_ADAGRAD ? mom_ptr(td, e) : nullptr,
                        reinterpret_cast<float4*>(row_ptr(td, e)));
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
// Warp per 32-position chunk.  Lane j owns position j's key, sample and
// table column; head/tail flags come from the neighbouring keys.  Rows are
// gathered U at a time and folded into a segmented running sum (reset to
// +0.0f at heads).  Pieces that end inside the chunk and started inside it
// are complete segments: their sums are staged in shared memory and the
// batch is updated together.  Edge pieces go to the level-2 buffer.
template <int VPL, int U>
__global__ void __launch_bounds__(kBwdThreads, 2) bwd_chunk_kernel(BwdArgs a) {
  __shared__ TabSmem ts;
  extern __shared__ float4 stage_mem[];  // [warps][U][32*VPL]
  const TabView tv = load_tables(a, ts);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4* stage = stage_mem + size_t(w) * U * 32 * VPL;
  const uint64_t nchunks = (a.L + kChunk - 1) / kChunk;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t c = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < nchunks; c += nwarps) {
    const uint64_t c0 = c * kChunk;
    const uint32_t n = uint32_t(min(uint64_t(kChunk), a.L - c0));
    const bool valid = uint32_t(lane) < n;
    const uint32_t k = valid ? a.keys[c0 + lane] : 0xFFFFFFFFu;
    const uint32_t b = valid ? a.vals[c0 + lane] : 0u;
    const uint32_t key_before = c0 > 0 ? a.keys[c0 - 1] : 0xFFFFFFFFu;
    const uint32_t key_after = c0 + n < a.L ? a.keys[c0 + n] : 0xFFFFFFFFu;
    uint32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
    uint32_t kn = __shfl_down_sync(0xffffffffu, k, 1);
    if (lane == 0) kp = key_before;
    if (uint32_t(lane) == n - 1) kn = key_after;
    const unsigned heads = __ballot_sync(0xffffffffu, valid && k != kp);
    const unsigned tails = __ballot_sync(0xffffffffu, valid && k != kn);
    // per-lane table (warp-uniform fast path when the chunk sits in one table)
    const uint32_t k0 = __shfl_sync(0xffffffffu, k, 0);
    const uint32_t kl = __shfl_sync(0xffffffffu, k, n - 1);
    uint32_t t = tv.find(k0);
    if (kl >= tv.kb[t + 1]) t = valid ? tv.find(k) : t;
    const uint32_t col = tv.col[t];
    const uint32_t dimv = tv.dim[t];
    float4 acc[VPL];
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) acc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t jb = 0; jb < n; jb += U) {
      float4 v[U][VPL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t pos = jb + u;
        const uint32_t bu = __shfl_sync(0xffffffffu, b, pos & 31);
        const uint32_t cu = __shfl_sync(0xffffffffu, col, pos & 31);
        const uint32_t Vu = __shfl_sync(0xffffffffu, dimv, pos & 31) >> 2;
        const float4* gr = reinterpret_cast<const float4*>(a.grad + uint64_t(bu) * a.stride + cu);
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) {
          const uint32_t vec = lane + vv * 32;
          v[u][vv] = (pos < n && vec < Vu) ? ld_nc_f4(gr + vec) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      int ns = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t pos = jb + u;
        if (pos < n) {
          if ((heads >> pos) & 1u) {
#pragma unroll
            for (int vv = 0; vv < VPL; ++vv) acc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) add4(acc[vv], v[u][vv]);
          if ((tails >> pos) & 1u) {
            const uint32_t Vu = __shfl_sync(0xffffffffu, dimv, pos) >> 2;
            if ((heads & (0xFFFFFFFFu >> (31 - pos))) == 0) {
              // began before this chunk, ends here: head edge piece
              store_vec<VPL>(a.part + (c * 2) * a.dmax, Vu, acc);
            } else {
#pragma unroll
              for (int vv = 0; vv < VPL; ++vv)
                if (uint32_t(lane + vv * 32) < Vu) stage[ns * 32 * VPL + lane + vv * 32] = acc[vv];
              ++ns;
            }
          }
        }
      }
      // keys / tables of the staged complete segments (in position order)
      if (ns) {
        const unsigned bm = (tails >> jb) & ((U >= 32) ? 0xFFFFFFFFu : ((1u << U) - 1u));
        // drop a leading head-edge piece (it was not staged)
        const unsigned upto = bm;
        unsigned staged = 0;
        int s = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t pos = jb + u;
          if (((upto >> u) & 1u) && (heads & (0xFFFFFFFFu >> (31 - pos))) != 0) staged |= 1u << u;
        }
        // lane s (< ns) takes the s-th staged position
        uint32_t my_pos = 0;
        unsigned rem = staged;
        for (s = 0; s < ns; ++s) {
          const int u = __ffs(rem) - 1;
          rem &= rem - 1;
          if (lane == s) my_pos = jb + u;
        }
        const uint32_t my_key = __shfl_sync(0xffffffffu, k, my_pos & 31);
        const uint32_t my_t = __shfl_sync(0xffffffffu, t, my_pos & 31);
        int32_t my_e = 0;
        if (lane < ns) {
          const TableDev& td = a.tables[my_t];
          my_e = td.remap[my_key - td.key_base];
        }
        // issue every row / state load of the batch, then update
        float4 wv[U][VPL];
        float mom[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int32_t e = __shfl_sync(0xffffffffu, my_e, q);
          const uint32_t tq = __shfl_sync(0xffffffffu, my_t, q);
          if (q < ns) {
            const TableDev& td = a.tables[tq];
            const float4* wp = reinterpret_cast<const float4*>(row_ptr(td, e));
#pragma unroll
            for (int vv = 0; vv < VPL; ++vv) {
              const uint32_t vec = lane + vv * 32;
              wv[q][vv] = vec < (td.dim >> 2) ? wp[vec] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            mom[q] = a.opt == RS_OPT_ROWWISE_ADAGRAD ? *mom_ptr(td, e) : 0.f;
          }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int32_t e = __shfl_sync(0xffffffffu, my_e, q);
          const uint32_t tq = __shfl_sync(0xffffffffu, my_t, q);
          if (q < ns) {
            const TableDev& td = a.tables[tq];
            float4 g[VPL];
#pragma unroll
            for (int vv = 0; vv < VPL; ++vv) g[vv] = stage[q * 32 * VPL + lane + vv * 32];
            update_row<VPL>(a, td.dim, g, wv[q], mom[q],
                            a.opt == RS_OPT_ROWWISE_ADAGRAD ? mom_ptr(td, e) : nullptr,
                            reinterpret_cast<float4*>(row_ptr(td, e)));
          }
        }
        __syncwarp();
      }
    }
    // the last piece continues into the next chunk: tail edge piece (or the
    // whole chunk is the middle of a segment: head edge piece)
    if (!((tails >> (n - 1)) & 1u)) {
      const uint32_t Vl = __shfl_sync(0xffffffffu, dimv, n - 1) >> 2;
      store_vec<VPL>(a.part + (c * 2 + (heads == 0 ? 0 : 1)) * a.dmax, Vl, acc);
    }
  }
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
        const uint32_t kk = slot == 0 ? f0 : f1;
        float4 x[VPL];
        if (!open || kk != run) {
          close();
          run = kk;
          open = true;
          t = tv.find(kk);
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
    if (a.keys[P1] != kl) continue;                                    // ends inside
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
