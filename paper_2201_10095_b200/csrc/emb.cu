// HP2 — the tiered EmbeddingBag operator that serves a RecShard plan.
//
// No reference implementation exists (the paper ran FBGEMM); the
// semantics follow the paper: sum-pool with an empty bag pooling to 0
// (PAPER.md:275), fast and slow tier rows read inside the same kernel
// (PAPER.md:605-607), the remap applied as part of the lookup (
// encoding include/shardplan/remap.hpp:27-29).  The forward's fast/slow hit
// counters equal simulate()'s accounting (core/src/simulator.cpp:86).
//
// HBM layout: per table a fast-tier block [hbm_rows, dim] (fp32 or fp16
// rows) in one device pool, the backed slow-tier block [slow_rows, dim] in one
// pinned, mapped host pool (read zero-copy over PCIe, or staged into HBM slots
// by uvm_cache.cuh), the int32 remap [hash_size] in HBM, and for row-wise
// Adagrad one fp32 state per row (both tiers' states in HBM).
//
// K4 forward: resolve_kernel turns every lookup's index into its storage-slot
//   key (remap applied; the backward's sort input) at streaming rate, then
//   forward_kernel runs a G-lane group per bag (G = lanes to cover dim/4
//   four-element vectors, <= 32), 32/G bags per warp-iteration; lanes load G
//   slot keys in parallel, then each group keeps 2 row gathers
//   (ld.global.nc) in flight and adds them in lookup order.
//   Warps claim 2 consecutive bag-groups at a time (the GPU sweeps the tables
//   in a narrow band); the next bag's offsets, first indices and remap
//   entries are prefetched behind the current bag's rows.
// K5 backward (emb_bwd.cuh): (slot key, sample) pairs written by the forward
//   -> per-table onesweep radix sort (scan_sort.cuh) -> segment descriptors ->
//   short segments (<= 32 lookups) summed in order and updated by G-lane
//   groups; long ones as 32-position pieces, 64-piece groups, then the row
//   update.  Fully deterministic, no float atomics.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <tuple>

#include <sys/mman.h>

#include "../../include/shardplan_gpu.h"
#include "context.cuh"
#include "exchange.cuh"
#include "host_worker.hpp"

namespace rs {
namespace emb {

struct TableDev {
  const int32_t* remap;
  char* fast;        // [hbm_rows][rbytes]
  char* slow;        // [slow_rows][rbytes], device view of pinned host memory
  float* mom_fast;
  float* mom_slow;
  const char* zero;  // one zero row (>= rbytes): what an unbacked row reads as
  uint64_t hash_size;
  uint64_t col;      // column offset in pooled rows
  uint32_t dim;
  uint32_t rbytes;   // dim * elem_bytes
  uint32_t ebytes;   // 4 (fp32) or 2 (fp16 storage, fp32 arithmetic)
  uint32_t nkeys;    // hbm_rows + slow_rows: the backward's key of every unbacked row
  uint64_t hbm_rows;
  uint64_t slow_rows;  // BACKED slow rows; slow offsets past them are unbacked
  // HBM staging of slow-tier rows (uvm_cache.cuh); slot_of == nullptr means
  // slow rows are read/written zero-copy in host memory.
  uint32_t* slot_of;
  char* staging;
  uint64_t stage_stride;  // bytes per staging slot
  // bit r: row r is a backed slow row (what the claim stages).  ceil(H/32)
  // words, L2-resident for a whole table set (RM1: 29 MB), so the claim
  // reads a row's remap entry only for the ~1% of lookups that are slow
  const uint32_t* sbits;
};

__host__ __device__ inline int lanes_for(uint32_t dim) {
  uint32_t v = dim / 4, L = 1;
  while (L < v && L < 32) L <<= 1;
  return int(L);
}

// Storage element <-> fp32, four at a time (a lane's `vec`: elements
// 4*vec .. 4*vec+3 of a row).  fp16 rows: 8-byte loads, exact widening,
// round-to-nearest-even narrowing on store.
template <class E>
struct Elem;
template <>
struct Elem<float> {
  using Raw = float4;  // a lane's four stored elements, as loaded
  static __device__ __forceinline__ Raw load_raw_nc(const char* row, uint32_t vec) {
    return ld_nc_f4(reinterpret_cast<const float4*>(row) + vec);
  }
  static __device__ __forceinline__ float4 widen_raw(Raw r) { return r; }
  static __device__ __forceinline__ Raw zero_raw() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  static __device__ __forceinline__ float4 load_nc(const char* row, uint32_t vec) {
    return ld_nc_f4(reinterpret_cast<const float4*>(row) + vec);
  }
  static __device__ __forceinline__ float4 load(const char* row, uint32_t vec) {
    return reinterpret_cast<const float4*>(row)[vec];
  }
  static __device__ __forceinline__ void store(char* row, uint32_t vec, float4 v) {
    reinterpret_cast<float4*>(row)[vec] = v;
  }
};
template <>
struct Elem<__half> {
  using Raw = uint2;
  static __device__ __forceinline__ Raw load_raw_nc(const char* row, uint32_t vec) {
    return ld_nc_u2(reinterpret_cast<const uint2*>(row) + vec);
  }
  static __device__ __forceinline__ Raw zero_raw() { return make_uint2(0u, 0u); }
  static __device__ __forceinline__ float4 widen(uint2 u) {
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
  static __device__ __forceinline__ float4 widen_raw(Raw r) { return widen(r); }
  static __device__ __forceinline__ float4 load_nc(const char* row, uint32_t vec) {
    return widen(ld_nc_u2(reinterpret_cast<const uint2*>(row) + vec));
  }
  static __device__ __forceinline__ float4 load(const char* row, uint32_t vec) {
    return widen(reinterpret_cast<const uint2*>(row)[vec]);
  }
  static __device__ __forceinline__ void store(char* row, uint32_t vec, float4 v) {
    const __half2 a = __floats2half2_rn(v.x, v.y), b = __floats2half2_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&a);
    u.y = *reinterpret_cast<const uint32_t*>(&b);
    reinterpret_cast<uint2*>(row)[vec] = u;
  }
};
// Runtime-typed access for the cold paths (init, read-back, long segments).
__device__ __forceinline__ float4 load4(const TableDev& td, const char* row, uint32_t vec) {
  return td.ebytes == 2 ? Elem<__half>::load(row, vec) : Elem<float>::load(row, vec);
}
__device__ __forceinline__ void store4(const TableDev& td, char* row, uint32_t vec, float4 v) {
  if (td.ebytes == 2) Elem<__half>::store(row, vec, v);
  else Elem<float>::store(row, vec, v);
}

// Slow offset of a (negative) remap entry.
__device__ __forceinline__ uint64_t slow_off(int32_t e) { return uint64_t(-int64_t(e) - 1); }
// Row of remap entry e in the host tier (no staging); unbacked rows read as zero.
__device__ __forceinline__ const char* row_ptr_host(const TableDev& td, int32_t e) {
  if (e >= 0) return td.fast + uint64_t(e) * td.rbytes;
  const uint64_t s = slow_off(e);
  return s < td.slow_rows ? td.slow + s * td.rbytes : td.zero;
}
// Row of remap entry e as the hot paths see it: slow rows come from their HBM
// staging slot when the batch was prefetched (uvm_cache.cuh).
// A slow row without a slot (a claim that ran out of slots: slot_of stays
// kNoSlot, 0xFFFFFFFF) is read/written in the host tier instead, so a failed
// claim can never send the kernels outside the staging buffer; the failure
// itself is reported before the batch runs (begin_step).  A slow offset past
// the backed rows (an omit_unaccessed remap, inc/remap.hpp:43-48) has no
// storage: it reads as the zero row and is never written (its backward key
// is the sentinel nkeys).
__device__ __forceinline__ char* row_ptr(const TableDev& td, int32_t e) {
  if (e >= 0) return td.fast + uint64_t(e) * td.rbytes;
  const uint64_t s = slow_off(e);
  if (s >= td.slow_rows) return const_cast<char*>(td.zero);
  if (td.slot_of) {
    const uint32_t sl = td.slot_of[s];
    if (sl < 0xFFFFFFFEu) return td.staging + uint64_t(sl) * td.stage_stride;
  }
  return td.slow + s * td.rbytes;
}
// The fast tier's base and row size held in registers for a hot loop (the
// compiler otherwise re-reads them from the table array for every row: stores
// elsewhere in the loop may alias it); slow rows take row_ptr.
struct RowBase {
  char* fast;
  uint32_t rbytes;
};
__device__ __forceinline__ RowBase row_base(const TableDev& td) { return RowBase{td.fast, td.rbytes}; }
__device__ __forceinline__ char* row_ptr(const TableDev& td, const RowBase& rb, int32_t e) {
  if (e >= 0) return rb.fast + uint64_t(uint32_t(e)) * rb.rbytes;
  return row_ptr(td, e);
}
__device__ __forceinline__ float* mom_ptr(const TableDev& td, int32_t e) {
  return e >= 0 ? td.mom_fast + uint64_t(e) : td.mom_slow + slow_off(e);
}
// Backward keys are storage slots within the table: key = e >= 0 ? e :
// hbm_rows + (-e - 1), a bijection of the backed remap entries onto
// [0, nkeys); every unbacked entry keys to nkeys (one segment per table that
// the update skips).  Tables keep their CSR position ranges (the backward
// sorts each table's range on its own).
__device__ __forceinline__ uint32_t slot_of_entry(const TableDev& td, int32_t e) {
  return e >= 0 ? uint32_t(e) : uint32_t(min(td.hbm_rows + slow_off(e), uint64_t(td.nkeys)));
}
__device__ __forceinline__ int32_t entry_of_key(const TableDev& td, uint32_t key) {
  const uint32_t s = key;
  return s < td.hbm_rows ? int32_t(s) : int32_t(-int64_t(s - td.hbm_rows) - 1);
}

constexpr int kFwdThreads = 256;

// Flushes a warp's accumulated (fast, total) lookup counts for table t (the
// caller's simulate() accounting, may be null) and its unbacked-row lookups.
__device__ __forceinline__ void flush_hits(unsigned long long* hits, unsigned long long* unbacked, uint32_t t,
                                           uint32_t fast, uint32_t tot, uint32_t unb) {
#pragma unroll
  for (int o2 = 16; o2; o2 >>= 1) {
    fast += __shfl_xor_sync(0xffffffffu, fast, o2);
    tot += __shfl_xor_sync(0xffffffffu, tot, o2);
    unb += __shfl_xor_sync(0xffffffffu, unb, o2);
  }
  if ((threadIdx.x & 31) == 0) {
    if (hits && tot) {
      atomicAdd(&hits[2 * uint64_t(t)], (unsigned long long)fast);
      atomicAdd(&hits[2 * uint64_t(t) + 1], (unsigned long long)(tot - fast));
    }
    if (unb) atomicAdd(&unbacked[t], (unsigned long long)unb);
  }
}

// Pipelined-bag helpers of forward_kernel: the bag's first G indices and
// their (checked) remap entries.
__device__ __forceinline__ uint32_t fwd_bag_index(const uint32_t* __restrict__ indices, int lg, uint32_t s,
                                                  uint32_t e) {
  return s < e && uint32_t(lg) < e - s ? ld_stream_u32(indices + s + lg) : 0u;
}
template <bool FK = false>
__device__ __forceinline__ int32_t fwd_bag_entry(const TableDev* __restrict__ tables, unsigned* err, int lg,
                                                 uint32_t t, uint32_t s, uint32_t e, uint32_t idx) {
  if (s >= e || uint32_t(lg) >= e - s) return 0;
  if (FK) return entry_of_key(tables[t], idx);
  const TableDev& tn = tables[t];
  if (idx >= tn.hash_size) {  // reported by the next backward / rs_emb_check
    atomicOr(err, 1u);
    idx = 0;
  }
  return tn.remap[idx];
}

// K4: a G-lane group per bag (BPW = 32/G bags per warp-iteration, a
// "bag-group"), software-pipelined over the warp's bags: the next bag's
// offsets are loaded at the top of this one, its first G indices once this
// bag's first row loads are in flight, and their remap entries once those
// rows have arrived — so a bag's dependent chain is its row loads, not
// offsets -> index -> remap -> rows.
//
// Scheduling: a warp claims `chunk` consecutive bag-groups (one atomic per
// chunk, the next chunk claimed a chunk ahead) and walks them in order with
// 32-bit incremental (table, bag) bookkeeping.  Small chunks keep the whole
// GPU inside a narrow band of one table's bags, so the table's Zipf head
// stays hot in L1/L2 (measured on B200, RM1: chunk 1 1.68 ms (counter
// contention), 2 1.30, 4 1.44, 16 2.03, 64 4.68; the old grid-stride loop
// 1.55 ms), and the per-table hit counters are flushed only when the table
// changes.
// FK: `indices` are the slot keys resolve_kernel wrote (entry_of_key instead
// of the remap load; the keys/vals for the backward are already written).
template <int G, int VPL, int UNR, int MINB, class E, bool FULL, bool FK = false>
__global__ void __launch_bounds__(kFwdThreads, MINB)
forward_kernel(const TableDev* __restrict__ tables, const uint32_t* __restrict__ cls_tables,
                uint32_t ntab, uint32_t B, const uint32_t* __restrict__ offsets,
                const uint32_t* __restrict__ indices, const OutMap om, uint64_t stride,
                unsigned long long* __restrict__ hits, unsigned long long* __restrict__ unbacked,
                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint64_t max_keys,
                unsigned* __restrict__ err, uint32_t* __restrict__ work, uint32_t chunk) {
  constexpr int BPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, lg = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const uint32_t wpt = (B + BPW - 1) / BPW;  // bag-groups per table
  const uint32_t total_w = wpt * ntab;
  auto grab = [&]() {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(work, 1u);
    return __shfl_sync(0xffffffffu, c, 0);
  };
  uint32_t cur_t = 0xFFFFFFFFu, fast = 0, tot = 0, unb = 0;
  // cursor: w (linear bag-group), wend (its chunk's end), ti / k (table slot,
  // bag-group within the table); cn: the chunk claimed ahead
  uint32_t w = grab() * chunk;
  if (w >= total_w) return;
  uint32_t wend = min(total_w, w + chunk);
  uint32_t ti = w / wpt, k = w - ti * wpt;
  uint32_t cn = grab();
  auto bag_offsets = [&](uint32_t ti_, uint32_t k_, uint32_t& t_, uint32_t& s_, uint32_t& e_) {
    t_ = cls_tables[ti_];
    const uint32_t bb = k_ * BPW + grp;
    s_ = e_ = 0;
    if (bb < B) {
      const uint64_t o = uint64_t(t_) * B + bb;
      s_ = offsets[o];
      e_ = offsets[o + 1];
    }
  };
  uint32_t nt = 0, ns = 0, ne = 0, nidx = 0;
  int32_t nent = 0;
  bag_offsets(ti, k, nt, ns, ne);
  nidx = fwd_bag_index(indices, lg, ns, ne);
  nent = fwd_bag_entry<FK>(tables, err, lg, nt, ns, ne, nidx);
  while (true) {
    const uint32_t t = nt, s = ns, e = ne;
    const int32_t ent0 = nent;
    const uint32_t kb = k;
    // advance the cursor to the next bag-group
    bool more = true;
    if (w + 1 < wend) {
      ++w;
      if (++k == wpt) {
        k = 0;
        ++ti;
      }
    } else {
      w = cn * chunk;
      if (w < total_w) {
        wend = min(total_w, w + chunk);
        ti = w / wpt;
        k = w - ti * wpt;
        cn = grab();
      } else {
        more = false;
      }
    }
    if (more) bag_offsets(ti, k, nt, ns, ne);
    bool pf = !more;  // next bag's index/entry issued?
    if (t != cur_t) {
      if (cur_t != 0xFFFFFFFFu) flush_hits(hits, unbacked, cur_t, fast, tot, unb);
      fast = tot = unb = 0;
      cur_t = t;
    }
    const TableDev& td = tables[t];
    const uint32_t V = td.dim >> 2;
    const RowBase rbase = row_base(td);
    const uint32_t b = kb * BPW + grp;
    const bool valid = b < B;
    float4 acc[VPL];
#pragma unroll
    for (int vv = 0; vv < VPL; ++vv) acc[vv] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lg == 0) {
      if (e > s) tot += e - s;
      else if (e < s) atomicOr(err, 16u);  // decreasing offsets: the next backward raises
    }
    for (uint32_t base = s; base < e; base += G) {
      const uint32_t n = min(uint32_t(G), e - base);
      int32_t ent = 0;
      if (uint32_t(lg) < n) {
        const uint32_t l = base + lg;
        if (base == s) {
          ent = ent0;
        } else {
          uint32_t idx = ld_stream_u32(indices + l);
          if (FK) {
            ent = entry_of_key(td, idx);
          } else {
            if (idx >= td.hash_size) {
              atomicOr(err, 1u);
              idx = 0;
            }
            ent = td.remap[idx];
          }
        }
        fast += ent >= 0;
        unb += ent < 0 && slow_off(ent) >= td.slow_rows;
        if (!FK && keys) {
          if (l < max_keys) {
            keys[l] = slot_of_entry(td, ent);
            vals[l] = b;
          } else {
            atomicOr(err, 2u);
          }
        }
      }
      // the bag's first block (up to UNR rows, predicated) carries the next
      // bag's prefetch: its first indices behind these row loads, their remap
      // entries after the adds; then whole blocks of UNR (no per-row
      // predicate) and the tail.  FULL (every table of the class exactly
      // G*VPL*4 wide) drops the per-lane width test.
      uint32_t j = 0;
      if (!pf) {
        float4 v[UNR][VPL];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int32_t eu = __shfl_sync(gmask, ent, u, G);
          const char* row = row_ptr(td, rbase, eu);
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) {
            const uint32_t vec = lg + vv * G;
            v[u][vv] = (uint32_t(u) < n && (FULL || vec < V)) ? Elem<E>::load_nc(row, vec)
                                                              : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        nidx = fwd_bag_index(indices, lg, ns, ne);
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          if (uint32_t(u) < n) {
#pragma unroll
            for (int vv = 0; vv < VPL; ++vv) {
              acc[vv].x = __fadd_rn(acc[vv].x, v[u][vv].x);
              acc[vv].y = __fadd_rn(acc[vv].y, v[u][vv].y);
              acc[vv].z = __fadd_rn(acc[vv].z, v[u][vv].z);
              acc[vv].w = __fadd_rn(acc[vv].w, v[u][vv].w);
            }
          }
        }
        nent = fwd_bag_entry<FK>(tables, err, lg, nt, ns, ne, nidx);
        pf = true;
        j = min(uint32_t(UNR), n);
      }
      for (; j + UNR <= n; j += UNR) {
        float4 v[UNR][VPL];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int32_t eu = __shfl_sync(gmask, ent, int(j) + u, G);
          const char* row = row_ptr(td, rbase, eu);
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) {
            const uint32_t vec = lg + vv * G;
            v[u][vv] = (FULL || vec < V) ? Elem<E>::load_nc(row, vec) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
#pragma unroll
          for (int vv = 0; vv < VPL; ++vv) {
            acc[vv].x = __fadd_rn(acc[vv].x, v[u][vv].x);
            acc[vv].y = __fadd_rn(acc[vv].y, v[u][vv].y);
            acc[vv].z = __fadd_rn(acc[vv].z, v[u][vv].z);
            acc[vv].w = __fadd_rn(acc[vv].w, v[u][vv].w);
          }
        }
      }
      for (; j < n; ++j) {
        const int32_t eu = __shfl_sync(gmask, ent, int(j), G);
        const char* row = row_ptr(td, rbase, eu);
        float4 v[VPL];
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) {
          const uint32_t vec = lg + vv * G;
          v[vv] = (FULL || vec < V) ? Elem<E>::load_nc(row, vec) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int vv = 0; vv < VPL; ++vv) {
          acc[vv].x = __fadd_rn(acc[vv].x, v[vv].x);
          acc[vv].y = __fadd_rn(acc[vv].y, v[vv].y);
          acc[vv].z = __fadd_rn(acc[vv].z, v[vv].z);
          acc[vv].w = __fadd_rn(acc[vv].w, v[vv].w);
        }
      }
    }
    if (!pf) {  // an empty bag: fetch the next one's head directly
      nidx = fwd_bag_index(indices, lg, ns, ne);
      nent = fwd_bag_entry<FK>(tables, err, lg, nt, ns, ne, nidx);
    }
    if (valid) {
      float4* o = reinterpret_cast<float4*>(out_row(om, b, stride) + (om.xcol ? om.xcol[t] : td.col));
#pragma unroll
      for (int vv = 0; vv < VPL; ++vv) {
        const uint32_t vec = lg + vv * G;
        if (FULL || vec < V) o[vec] = acc[vv];
      }
    }
    if (!more) break;
  }
  if (cur_t != 0xFFFFFFFFu) flush_hits(hits, unbacked, cur_t, fast, tot, unb);
}

// ------------------------------------------------------------------ backward
// keys[l] = storage slot of remap[index] in table t, vals[l] = sample b, for
// every lookup l of bag (t, b); warps flatten 32 bags' lookups so stores stay
// coalesced.  Keying by slot lets the backward address rows without a remap
// load and walks each tier in address order.
__global__ void __launch_bounds__(256)
keygen_kernel(const TableDev* __restrict__ tables, uint32_t T, uint64_t B,
              const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ indices,
              uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, unsigned* __restrict__ err) {
  if (*reinterpret_cast<volatile unsigned*>(err)) return;  // offsets rejected by bwd_plan_kernel
  const int lane = threadIdx.x & 31;
  const uint64_t nbags = uint64_t(T) * B;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t c = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c * 32 < nbags; c += nwarps) {
    const uint64_t g = c * 32 + lane;
    uint32_t s = 0, len = 0, t = 0;
    uint64_t H = 0;
    if (g < nbags) {
      s = offsets[g];
      const uint32_t e = offsets[g + 1];
      if (e < s) atomicOr(err, 16u);  // a decreasing bag: the gate empties the plan
      len = e > s ? e - s : 0u;
      t = uint32_t(g / B);
      H = tables[t].hash_size;
    }
    const uint32_t incl = warp_incl_scan(len);
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = incl - len;
    const uint32_t s0 = __shfl_sync(0xffffffffu, s, 0);
    for (uint32_t p = 0; p < total; p += 32) {
      const uint32_t q = p + lane;
      int k = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        uint32_t ex = __shfl_sync(0xffffffffu, excl, k + step);
        if (ex <= q) k += step;
      }
      const uint64_t Hk = __shfl_sync(0xffffffffu, H, k);
      const uint64_t gk = c * 32 + k;
      if (q < total) {
        const uint32_t l = s0 + q;  // bags are contiguous in table-major CSR
        const uint32_t idx = indices[l];
        if (idx >= Hk) atomicOr(err, 1u);
        const TableDev& tdk = tables[gk / B];
        keys[l] = slot_of_entry(tdk, tdk.remap[idx < Hk ? idx : 0u]);
        vals[l] = uint32_t(gk % B);
      }
    }
  }
}


// The forward's index resolution as its own streaming pass: for every lookup
// l of bag (t, b), keys[l] = storage slot of remap[indices[l]] and vals[l] =
// b (the backward's sort input).  A warp takes 32 consecutive bags, flattens
// their lookups over its lanes and keeps 4 lookups per lane in flight, so the
// index -> remap chain runs at streaming rate instead of on the gather's
// critical path; the gather then reads the slot keys (forward_kernel<FK>).
__global__ void __launch_bounds__(256)
resolve_kernel(const TableDev* __restrict__ tables, uint32_t T, uint32_t B, const uint32_t* __restrict__ offsets,
               const uint32_t* __restrict__ indices, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
               uint64_t max_keys, unsigned* __restrict__ err) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const uint64_t nbags = uint64_t(T) * B;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t c = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c * 32 < nbags; c += nwarps) {
    const uint64_t g = c * 32 + lane;
    uint32_t s = 0, len = 0, t = 0, b = 0;
    if (g < nbags) {
      s = offsets[g];
      const uint32_t e = offsets[g + 1];
      len = e > s ? e - s : 0u;  // decreasing offsets: flagged by the forward
      t = uint32_t(g / B);
      b = uint32_t(g - uint64_t(t) * B);
    }
    const uint32_t incl = warp_incl_scan(len);
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = incl - len;
    const uint32_t s0 = __shfl_sync(0xffffffffu, s, 0);
    for (uint32_t p = 0; p < total; p += 32 * U) {
      uint32_t id[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = p + uint32_t(u) * 32 + lane;
        id[u] = q < total ? ld_stream_u32(indices + s0 + q) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = p + uint32_t(u) * 32 + lane;
        int k = 0;  // the lookup's bag: the last lane whose range starts at or before q
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const uint32_t ex = __shfl_sync(0xffffffffu, excl, k + step);
          if (ex <= q) k += step;
        }
        const uint32_t tk = __shfl_sync(0xffffffffu, t, k);
        const uint32_t bk = __shfl_sync(0xffffffffu, b, k);
        if (q < total) {
          const uint32_t l = s0 + q;  // bags are contiguous in table-major CSR
          const TableDev& td = tables[tk];
          uint32_t idx = id[u];
          if (idx >= td.hash_size) {
            atomicOr(err, 1u);  // reported by the next backward / rs_emb_check
            idx = 0;
          }
          if (l < max_keys) {
            keys[l] = slot_of_entry(td, td.remap[idx]);
            vals[l] = bk;
          } else {
            atomicOr(err, 2u);
          }
        }
      }
    }
  }
}

}  // namespace emb
}  // namespace rs

#include "emb_bwd.cuh"
#include "uvm_cache.cuh"

namespace rs {
namespace emb {

// ------------------------------------------------------------------ init / read
// Init values are drawn in fp32 (or_init_weight) and rounded to the storage
// type; unbacked rows have no storage.
__global__ void init_kernel(TableDev td, uint32_t table_id, uint64_t seed, float scale) {
  const uint32_t V = td.dim >> 2;
  const uint64_t n = td.hash_size * V;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t row = i / V;
    const uint32_t vec = uint32_t(i % V);
    const int32_t e = td.remap[row];
    if (e < 0 && slow_off(e) >= td.slow_rows) continue;
    const uint64_t ds = derive_stream(seed, table_id, row);
    float x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t u = mix64(ds + vec * 4 + k) >> 40;
      x[k] = __fmul_rn(__fsub_rn(__fmul_rn(float(u), 0x1.0p-24f), 0.5f), scale);
    }
    store4(td, const_cast<char*>(row_ptr_host(td, e)), vec, make_float4(x[0], x[1], x[2], x[3]));
    if (vec == 0 && td.mom_fast) *mom_ptr(td, e) = 0.f;
  }
}

// Rows by original id, widened to fp32 (unbacked rows read as zero, momentum 0).
__global__ void read_rows_kernel(TableDev td, const uint32_t* __restrict__ rows, uint64_t n,
                                 float* __restrict__ out, float* __restrict__ mom_out) {
  const uint32_t V = td.dim >> 2;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n * V;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / V;
    const uint32_t vec = uint32_t(i % V);
    const int32_t e = td.remap[rows[r]];
    const bool backed = e >= 0 || slow_off(e) < td.slow_rows;
    reinterpret_cast<float4*>(out + r * td.dim)[vec] = load4(td, row_ptr_host(td, e), vec);
    if (mom_out && vec == 0) mom_out[r] = td.mom_fast && backed ? *mom_ptr(td, e) : 0.f;
  }
}

// Every remap entry must land inside its tier: fast entries below hbm_rows,
// slow ones below slow_rows unless unbacked rows are allowed (then anything
// past slow_rows is an unbacked row and counted).
// Slow-row bitmap of one table (TableDev::sbits), a warp ballot per 32 rows.
__global__ void slow_bits_kernel(const int32_t* __restrict__ remap, uint64_t H, uint64_t slow_rows,
                                 uint32_t* __restrict__ bits) {
  const uint64_t nw = (H + 31) / 32;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < nw; w += nwarps) {
    const uint64_t r = w * 32 + (threadIdx.x & 31);
    const int32_t e = r < H ? remap[r] : 0;
    const uint32_t b = __ballot_sync(0xffffffffu, e < 0 && slow_off(e) < slow_rows);
    if ((threadIdx.x & 31) == 0) bits[w] = b;
  }
}

__global__ void check_remap_kernel(const int32_t* __restrict__ remap, uint64_t H, uint64_t hbm_rows,
                                   uint64_t slow_rows, int allow_unbacked, unsigned* __restrict__ err,
                                   unsigned long long* __restrict__ n_unbacked) {
  uint32_t unb = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < H;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const int32_t e = remap[i];
    if (e >= 0) {
      if (uint64_t(e) >= hbm_rows) atomicOr(err, 1u);
    } else if (slow_off(e) >= slow_rows) {
      if (allow_unbacked) ++unb;
      else atomicOr(err, 1u);
    }
  }
  if (unb) atomicAdd(n_unbacked, (unsigned long long)unb);
}

}  // namespace emb
}  // namespace rs

using rs::emb::TableDev;

struct rs_emb {
  rs_context* ctx = nullptr;
  uint32_t T = 0;
  uint64_t max_batch = 0, max_lookups = 0;
  int opt = RS_OPT_SGD;
  float eps = 1e-8f;
  std::vector<TableDev> h_tables;
  std::vector<uint32_t> table_ids;
  TableDev* d_tables = nullptr;
  uint64_t total_dim = 0;
  uint32_t dmax = 0;
  uint32_t rmax = 0;  // max row bytes (staging slot stride)
  char* fast_pool = nullptr;
  size_t fast_bytes = 0;
  char* host_pool = nullptr;
  char* host_pool_dev = nullptr;
  bool host_mapped = false;  // mmap + THP + cudaHostRegister (else cudaHostAlloc)
  void* host_map_base = nullptr;
  size_t host_map_bytes = 0;
  size_t host_bytes = 0;
  int32_t* remap_pool = nullptr;
  uint32_t* sbits_pool = nullptr;  // TableDev::sbits of every table
  size_t remap_bytes = 0;
  // unbacked rows (omit_unaccessed remaps): per-table lookup counters, the
  // zero row they read, and how many remap entries each table leaves unbacked
  unsigned long long* d_unbacked = nullptr;
  uint32_t* d_work = nullptr;  // forward_kernel's chunk counters (one per lane class)
  bool resolved = false;       // the running forward's keys come from resolve_kernel
  char* zero_row = nullptr;
  std::vector<uint64_t> unbacked_rows;
  // forward classes: (G, VPL, element bytes) -> table list
  struct Class {
    int G, VPL, EB;
    std::vector<uint32_t> tables;
    uint32_t* d_list = nullptr;
    bool full = true;  // every table exactly 4*G*VPL wide (no per-lane width test)
  };
  std::vector<Class> classes;
  uint32_t key_bits = 0;  // max over tables of the slot-key width
  // segmented sort tiles (per table): pos[ntiles+1] | cidx[ntiles] | cstride[ntiles]
  uint32_t* d_tiles = nullptr;
  size_t tiles_cap = 0;
  int bwd_vpl = 1;
  // backward buffers
  uint32_t* keys = nullptr;
  uint32_t* vals = nullptr;
  // the last forward wrote (keys, vals) for its batch: a backward of the same
  // (offsets, indices, batch) skips keygen
  const uint32_t* keys_off = nullptr;
  const uint32_t* keys_idx = nullptr;
  uint64_t keys_B = 0;
  // HBM staging of slow rows (uvm_cache.cuh)
  uint32_t nslots = 0;
  char* staging = nullptr;
  uint32_t* slot_of = nullptr;  // sum(slow_rows)
  uint32_t* slot_gen = nullptr;
  uint32_t* slot_tab = nullptr;
  uint32_t* slot_row = nullptr;
  uint32_t* free_stack = nullptr;
  uint32_t* copy_list = nullptr;
  int* free_top = nullptr;
  unsigned* ncopy = nullptr;
  unsigned* cache_err = nullptr;
  // DMA staging (uvm_cache.cuh): bounce buffers of bcap rows (stride dmax)
  uint32_t bcap = 0;
  uint32_t *copy_tab = nullptr, *copy_row = nullptr, *wb_tab = nullptr, *wb_row = nullptr;
  unsigned* n_wb = nullptr;
  char *d_bin = nullptr, *d_bout = nullptr, *h_bin = nullptr, *h_bout = nullptr;
  uint32_t *h_ctab = nullptr, *h_crow = nullptr, *h_wtab = nullptr, *h_wrow = nullptr;
  unsigned* h_cnt = nullptr;
  cudaEvent_t ev_claim[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_evict[4] = {nullptr, nullptr, nullptr, nullptr};  // ring: one per eviction in flight
  std::vector<cudaEvent_t> ev_out_chunk;  // stage-out: one per D2H chunk (grown on demand, out worker only)
  uint64_t n_evicts = 0;
  cudaEvent_t last_claim = nullptr;  // the most recent claim (side stream)
  std::unique_ptr<rs::TaskQueue> worker;      // stage-in tasks (host tier -> slots)
  std::unique_ptr<rs::TaskQueue> out_worker;  // stage-out tasks (evicted rows -> host tier)
  std::unique_ptr<rs::ThreadPool> pool, out_pool;
  cudaStream_t side_out = nullptr;
  cudaStream_t claim_stream = nullptr;
  uint64_t gather_seq[4] = {0, 0, 0, 0}, wb_seq = 0;
  unsigned gen_err[4] = {0, 0, 0, 0};  // cache_err seen by generation g's stage-in (host)
  // set by the exchange (exchange.cu) for one backward: the gradient rows it
  // reads are complete once this event has fired
  cudaEvent_t grad_ready = nullptr;

  TableDev* d_tables_c = nullptr;
  uint32_t* d_slow_tabs = nullptr;  // tables with slow rows
  uint32_t nslow_tabs = 0;
  const TableDev* cur_tables = nullptr;  // tables the running forward/backward use
  cudaStream_t side = nullptr;
  cudaEvent_t ev_main = nullptr, ev_gather[4] = {nullptr, nullptr, nullptr, nullptr};
  // kernel-only timing: event pairs around the forward / backward kernel
  // sequences (excluding staging waits), harvested by rs_emb_kernel_times
  struct Timer {
    static constexpr int kRing = 64;
    cudaEvent_t ev[kRing][2] = {};
    int n = 0;
    double ms = 0;
    uint64_t count = 0;
    void begin(cudaStream_t s) {
      if (n == kRing) harvest();
      if (!ev[n][0]) {
        RS_CUDA(cudaEventCreate(&ev[n][0]));
        RS_CUDA(cudaEventCreate(&ev[n][1]));
      }
      RS_CUDA(cudaEventRecord(ev[n][0], s));
    }
    void end(cudaStream_t s) { RS_CUDA(cudaEventRecord(ev[n++][1], s)); }
    void harvest() {
      for (int i = 0; i < n; ++i) {
        float t = 0;
        RS_CUDA(cudaEventSynchronize(ev[i][1]));
        RS_CUDA(cudaEventElapsedTime(&t, ev[i][0], ev[i][1]));
        ms += t;
        ++count;
      }
      n = 0;
    }
    ~Timer() {
      for (auto& p : ev)
        for (cudaEvent_t x : p)
          if (x) cudaEventDestroy(x);
    }
  } t_fwd, t_bwd;
  std::vector<uint64_t> pending;  // prefetched generations, oldest first
  int64_t cur_gen = -1;           // staged generation of the running step (-1: zero-copy)
  int64_t done_gen = -1;          // finished generation, evicted one step later
  uint64_t next_gen = 0;
  bool staged_dirty = false;
  uint32_t* scount = nullptr;  // [windows + 1] segment heads per window
  uint32_t* sbase = nullptr;   // [windows + 1] exclusive scan of scount
  uint4* segs = nullptr;       // [max_lookups] segment descriptors
  size_t long_cap = 0;         // long segments (> 32 positions) <= lookups / 33
  uint4* longs = nullptr;
  uint32_t* long_np = nullptr;  // [long_cap] first piece of each long segment
  uint32_t* long_ng = nullptr;  // [long_cap] first group of each long segment
  uint2* gdesc = nullptr;       // [groups] {long slot, group within it}
  unsigned* n_long = nullptr;   // {long slots, pieces, groups}
  float* ppart = nullptr;       // [pieces][dmax] piece sums of long segments
  uint4* pdesc = nullptr;       // [pieces] {start, count, table} of each piece
  float* gpart = nullptr;       // [groups][dmax] group sums of long segments
  uint32_t* d_meta = nullptr;
  uint32_t* h_meta = nullptr;
  size_t meta_words = 0;
  // device backward plan (bwd_plan_kernel): class-major table order, class
  // boundaries, class window bounds, sort tile count; the error word's copy
  uint32_t* d_order = nullptr;
  uint32_t* d_cpos = nullptr;
  uint32_t* d_cw = nullptr;
  uint32_t* d_nt = nullptr;
  cudaEvent_t ev_err = nullptr;
  cudaStream_t fwd_side = nullptr;  // every other forward lane class
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  unsigned* d_err = nullptr;
  char* sort_scratch = nullptr;
  size_t sort_scratch_bytes = 0;

  ~rs_emb() {
    worker.reset();  // joins the staging workers before any buffer goes
    out_worker.reset();
    pool.reset();
    out_pool.reset();
    for (cudaStream_t x : {side_out, claim_stream})
      if (x) {
        cudaStreamSynchronize(x);
        cudaStreamDestroy(x);
      }
    for (void* p : {(void*)h_bin, (void*)h_bout, (void*)h_ctab, (void*)h_crow, (void*)h_wtab, (void*)h_wrow,
                    (void*)h_cnt})
      if (p) cudaFreeHost(p);
    for (void* p : {(void*)copy_tab, (void*)copy_row, (void*)wb_tab, (void*)wb_row, (void*)n_wb, (void*)d_bin,
                    (void*)d_bout})
      if (p) cudaFree(p);
    for (cudaEvent_t ev : {ev_claim[0], ev_claim[1], ev_claim[2], ev_claim[3], ev_evict[0], ev_evict[1],
                           ev_evict[2], ev_evict[3]})
      if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : ev_out_chunk) cudaEventDestroy(ev);
    if (d_tables) cudaFree(d_tables);
    if (fast_pool) cudaFree(fast_pool);
    if (host_pool) {
      if (host_mapped) {
        cudaHostUnregister(host_pool);
        munmap(host_map_base, host_map_bytes);
      } else {
        cudaFreeHost(host_pool);
      }
    }
    if (remap_pool) cudaFree(remap_pool);
    if (sbits_pool) cudaFree(sbits_pool);
    for (auto& c : classes)
      if (c.d_list) cudaFree(c.d_list);
    if (d_tiles) cudaFree(d_tiles);
    if (keys) cudaFree(keys);
    if (vals) cudaFree(vals);
    for (void* p : {(void*)scount, (void*)sbase, (void*)segs, (void*)longs, (void*)long_np, (void*)long_ng,
                    (void*)gdesc, (void*)n_long, (void*)ppart, (void*)pdesc, (void*)gpart})
      if (p) cudaFree(p);
    if (d_meta) cudaFree(d_meta);
    if (h_meta) cudaFreeHost(h_meta);
    for (void* p : {(void*)d_order, (void*)d_cpos, (void*)d_cw, (void*)d_nt})
      if (p) cudaFree(p);
    if (ev_err) cudaEventDestroy(ev_err);
    for (cudaEvent_t ev : {ev_fork, ev_join})
      if (ev) cudaEventDestroy(ev);
    if (fwd_side) {
      cudaStreamSynchronize(fwd_side);
      cudaStreamDestroy(fwd_side);
    }
    if (d_err) cudaFree(d_err);
    for (void* p : {(void*)d_unbacked, (void*)zero_row, (void*)d_work})
      if (p) cudaFree(p);
    if (sort_scratch) cudaFree(sort_scratch);
    if (side) {
      cudaStreamSynchronize(side);
      cudaStreamDestroy(side);
    }
    for (cudaEvent_t ev : {ev_main, ev_gather[0], ev_gather[1], ev_gather[2], ev_gather[3]})
      if (ev) cudaEventDestroy(ev);
    for (void* p : {(void*)staging, (void*)slot_of, (void*)slot_gen, (void*)slot_tab, (void*)slot_row,
                    (void*)free_stack, (void*)copy_list, (void*)free_top, (void*)ncopy, (void*)cache_err,
                    (void*)d_tables_c, (void*)d_slow_tabs})
      if (p) cudaFree(p);
  }
};

namespace rs {

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// The pinned host tier.  Random row gathers/scatters over tens of GB miss the
// TLB on every row with 4 KiB pages, so the tier is an anonymous mapping
// advised for transparent huge pages (2 MiB) and then pinned and mapped with
// cudaHostRegister; cudaHostAlloc is the fallback (RS_HOST_THP=0 forces it).
static void alloc_host_tier(rs_emb* e) {
  const char* env = getenv("RS_HOST_THP");
  const bool thp = !(env && env[0] == '0');
  constexpr size_t kHuge = size_t(2) << 20;
  if (thp) {
    const size_t bytes = (e->host_bytes + kHuge - 1) / kHuge * kHuge;
    const size_t map = bytes + kHuge;
    void* base = mmap(nullptr, map, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (base != MAP_FAILED) {
      char* p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(base) + kHuge - 1) & ~uintptr_t(kHuge - 1));
      madvise(p, bytes, MADV_HUGEPAGE);
      if (cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
        e->host_pool = p;
        e->host_mapped = true;
        e->host_map_base = base;
        e->host_map_bytes = map;
        return;
      }
      cudaGetLastError();
      munmap(base, map);
    }
  }
  RS_CUDA(cudaHostAlloc(&e->host_pool, e->host_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
}

rs_emb* emb_create(rs_context* ctx, uint32_t T, const rs_emb_table* tabs, uint64_t max_batch,
                   uint64_t max_lookups, int opt, float eps) {
  using namespace emb;
  if (T == 0) throw InvalidArgument("emb: no tables");
  if (opt != RS_OPT_SGD && opt != RS_OPT_ROWWISE_ADAGRAD) throw InvalidArgument("emb: unknown optimizer");
  if (max_batch == 0) throw InvalidArgument("emb: max_batch must be >= 1");
  if (max_lookups >= (uint64_t(1) << 32)) throw InvalidArgument("emb: max_lookups must be < 2^32");
  auto* e = new rs_emb;
  e->ctx = ctx;
  // the context's scratch is transient; a large one (left by a profile of a
  // big table set) would otherwise crowd out the tiers allocated below
  if (ctx->arena_cap > (size_t(1) << 30)) ctx->trim_scratch();
  e->T = T;
  e->max_batch = max_batch;
  e->max_lookups = max_lookups;
  e->opt = opt;
  e->eps = eps;
  try {
    cudaStream_t st = ctx->stream;
    size_t fb = 0, hb = 0, rb = 0, sb = 0;
    std::vector<size_t> foff(T), hoff(T), roff(T), soff(T), mfoff(T), mhoff(T);
    std::vector<uint32_t> eb(T);
    for (uint32_t t = 0; t < T; ++t) {
      const rs_emb_table& x = tabs[t];
      if (x.dim == 0 || x.dim % 4 || x.dim > 1024)
        throw InvalidArgument("emb: table " + std::to_string(x.table_id) + ": dim must be a multiple of 4 in [4, 1024]");
      if (x.hash_size == 0 || x.hash_size > 0x7FFFFFFFULL)
        throw InvalidArgument("emb: table " + std::to_string(x.table_id) + ": hash_size out of range");
      if (x.hbm_rows > x.hash_size) throw InvalidArgument("emb: hbm_rows exceeds hash_size");
      if (x.hbm_rows + x.slow_rows > x.hash_size)
        throw InvalidArgument("emb: table " + std::to_string(x.table_id) + ": hbm_rows + slow_rows exceeds hash_size");
      if (!x.remap) throw InvalidArgument("emb: table " + std::to_string(x.table_id) + " has no remap");
      eb[t] = x.elem_bytes ? x.elem_bytes : 4u;
      if (eb[t] != 2 && eb[t] != 4)  // inc/types.hpp:50-52
        throw InvalidArgument("emb: table " + std::to_string(x.table_id) + ": elem_bytes must be 2 or 4");
      foff[t] = fb;
      fb += align256(x.hbm_rows * x.dim * eb[t]);
      hoff[t] = hb;
      hb += align256(x.slow_rows * x.dim * eb[t]);
      roff[t] = rb;
      rb += align256(x.hash_size * 4);
      soff[t] = sb;
      sb += align256((x.hash_size + 31) / 32 * 4);
      e->total_dim += x.dim;
      e->dmax = std::max(e->dmax, x.dim);
      e->rmax = std::max(e->rmax, (x.dim * eb[t] + 15) / 16 * 16);
      e->table_ids.push_back(x.table_id);
    }
    // Adagrad state (4 B/row) of BOTH tiers lives in HBM: a slow-tier row's
    // update then costs one PCIe row read + write instead of four transfers.
    if (opt == RS_OPT_ROWWISE_ADAGRAD) {
      for (uint32_t t = 0; t < T; ++t) {
        mfoff[t] = fb;
        fb += align256(tabs[t].hbm_rows * 4);
        mhoff[t] = fb;
        fb += align256(tabs[t].slow_rows * 4);
      }
    }
    e->fast_bytes = std::max<size_t>(fb, 256);
    e->host_bytes = std::max<size_t>(hb, 256);
    e->remap_bytes = rb;
    if (cudaMalloc(&e->fast_pool, e->fast_bytes) != cudaSuccess) {
      cudaGetLastError();
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      throw CudaError("emb: fast tier of " + std::to_string(e->fast_bytes >> 20) + " MiB does not fit (" +
                      std::to_string(fr >> 20) + " MiB free of " + std::to_string(tot >> 20) + ")");
    }
    alloc_host_tier(e);
    RS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->host_pool_dev), e->host_pool, 0));
    RS_CUDA(cudaMalloc(&e->remap_pool, std::max<size_t>(rb, 256)));
    RS_CUDA(cudaMalloc(&e->sbits_pool, std::max<size_t>(sb, 256)));
    RS_CUDA(cudaMalloc(&e->d_err, 16));
    RS_CUDA(cudaMalloc(&e->d_unbacked, 8 * size_t(T)));
    RS_CUDA(cudaMalloc(&e->d_work, 256));
    RS_CUDA(cudaMemsetAsync(e->d_unbacked, 0, 8 * size_t(T), st));
    RS_CUDA(cudaMalloc(&e->zero_row, 4096));
    RS_CUDA(cudaMemsetAsync(e->zero_row, 0, 4096, st));
    e->unbacked_rows.assign(T, 0);
    uint64_t col = 0;
    e->h_tables.resize(T);
    for (uint32_t t = 0; t < T; ++t) {
      const rs_emb_table& x = tabs[t];
      TableDev& d = e->h_tables[t];
      d.remap = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(e->remap_pool) + roff[t]);
      RS_CUDA(cudaMemcpyAsync(const_cast<int32_t*>(d.remap), x.remap, x.hash_size * 4,
                              x.remap_location == RS_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                                : cudaMemcpyHostToDevice,
                              st));
      d.sbits = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(e->sbits_pool) + soff[t]);
      {
        const unsigned gb = unsigned(std::max<uint64_t>(
            1, std::min<uint64_t>(((x.hash_size + 31) / 32 + 7) / 8, uint64_t(sm_count()) * 8)));
        slow_bits_kernel<<<gb, 256, 0, st>>>(d.remap, x.hash_size, x.slow_rows, const_cast<uint32_t*>(d.sbits));
        RS_COUNT(1);
      }
      d.fast = e->fast_pool + foff[t];
      d.slow = e->host_pool_dev + hoff[t];
      d.zero = e->zero_row;
      d.ebytes = eb[t];
      d.rbytes = x.dim * eb[t];
      d.nkeys = uint32_t(x.hbm_rows + x.slow_rows);
      d.mom_fast = opt == RS_OPT_ROWWISE_ADAGRAD ? reinterpret_cast<float*>(e->fast_pool + mfoff[t]) : nullptr;
      d.mom_slow = opt == RS_OPT_ROWWISE_ADAGRAD ? reinterpret_cast<float*>(e->fast_pool + mhoff[t]) : nullptr;
      d.hash_size = x.hash_size;
      d.col = col;
      d.dim = x.dim;
      d.hbm_rows = x.hbm_rows;
      d.slow_rows = x.slow_rows;
      col += x.dim;
      // every remap entry must land inside its tier's allocation
      RS_CUDA(cudaMemsetAsync(e->d_err, 0, 16, st));
      unsigned g = unsigned(std::min<uint64_t>((x.hash_size + 255) / 256, uint64_t(sm_count()) * 8));
      check_remap_kernel<<<std::max(1u, g), 256, 0, st>>>(d.remap, x.hash_size, x.hbm_rows, x.slow_rows,
                                                          x.allow_unbacked, e->d_err,
                                                          reinterpret_cast<unsigned long long*>(e->d_err + 2));
      unsigned herr[4] = {0, 0, 0, 0};
      RS_CUDA(cudaMemcpyAsync(herr, e->d_err, 16, cudaMemcpyDeviceToHost, st));
      RS_CUDA(cudaStreamSynchronize(st));
      if (herr[0])
        throw InvalidArgument("emb: table " + std::to_string(x.table_id) +
                              ": remap entry outside the fast/slow tier sizes");
      std::memcpy(&e->unbacked_rows[t], herr + 2, 8);
    }
    e->key_bits = 1;
    // keys span [0, nkeys] (nkeys: the unbacked sentinel)
    for (uint32_t t = 0; t < T; ++t) {
      const uint64_t nk = uint64_t(e->h_tables[t].nkeys) + (e->unbacked_rows[t] ? 1 : 0);
      while (e->key_bits < 32 && (uint64_t(1) << e->key_bits) < nk) ++e->key_bits;
    }
    RS_CUDA(cudaMalloc(&e->d_tables, sizeof(TableDev) * T));
    RS_CUDA(cudaMemcpyAsync(e->d_tables, e->h_tables.data(), sizeof(TableDev) * T, cudaMemcpyHostToDevice, st));
    // forward classes
    for (uint32_t t = 0; t < T; ++t) {
      const int G = lanes_for(tabs[t].dim);
      const int VPL = int((tabs[t].dim / 4 + G - 1) / G);
      int vp2 = 1;
      while (vp2 < VPL) vp2 <<= 1;
      const int EB = int(eb[t]);
      auto it = std::find_if(e->classes.begin(), e->classes.end(),
                             [&](const rs_emb::Class& c) { return c.G == G && c.VPL == vp2 && c.EB == EB; });
      if (it == e->classes.end()) {
        e->classes.push_back({G, vp2, EB, {}, nullptr, true});
        it = e->classes.end() - 1;
      }
      it->tables.push_back(t);
      if (tabs[t].dim != uint32_t(4 * G * vp2)) it->full = false;
    }
    for (auto& c : e->classes) {
      RS_CUDA(cudaMalloc(&c.d_list, 4 * c.tables.size()));
      RS_CUDA(cudaMemcpyAsync(c.d_list, c.tables.data(), 4 * c.tables.size(), cudaMemcpyHostToDevice, st));
    }
    {
      std::vector<uint32_t> order, cpos{0};
      for (auto& c : e->classes) {
        order.insert(order.end(), c.tables.begin(), c.tables.end());
        cpos.push_back(uint32_t(order.size()));
      }
      RS_CUDA(cudaMalloc(&e->d_order, 4 * std::max<size_t>(1, order.size())));
      RS_CUDA(cudaMalloc(&e->d_cpos, 4 * cpos.size()));
      RS_CUDA(cudaMalloc(&e->d_cw, 4 * cpos.size()));
      RS_CUDA(cudaMalloc(&e->d_nt, 4));
      if (!order.empty())
        RS_CUDA(cudaMemcpy(e->d_order, order.data(), 4 * order.size(), cudaMemcpyHostToDevice));
      RS_CUDA(cudaMemcpy(e->d_cpos, cpos.data(), 4 * cpos.size(), cudaMemcpyHostToDevice));
      RS_CUDA(cudaEventCreateWithFlags(&e->ev_err, cudaEventDisableTiming));
      RS_CUDA(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
      RS_CUDA(cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
      // the second forward lane runs at the caller stream's priority (the
      // staging streams keep the default, lowest one)
      int prio = 0;
      RS_CUDA(cudaStreamGetPriority(e->ctx->stream, &prio));
      RS_CUDA(cudaStreamCreateWithPriority(&e->fwd_side, cudaStreamNonBlocking, prio));
    }
    {
      int v = 1;
      while (v * 32 * 4 < int(e->dmax)) v <<= 1;
      e->bwd_vpl = v;
    }
    // backward buffers
    const size_t L = std::max<uint64_t>(max_lookups, 1);
    RS_CUDA(cudaMalloc(&e->keys, L * 4));
    RS_CUDA(cudaMalloc(&e->vals, L * 4));
    const size_t nch = (L + emb::kChunk - 1) / emb::kChunk + T;  // windows (per-table rounding)
    RS_CUDA(cudaMalloc(&e->scount, (nch + 1) * 4));
    RS_CUDA(cudaMalloc(&e->sbase, (nch + 1) * 4));
    RS_CUDA(cudaMalloc(&e->segs, L * sizeof(uint4)));
    e->long_cap = L / (emb::kChunk + 1) + 1;
    RS_CUDA(cudaMalloc(&e->longs, e->long_cap * sizeof(uint4)));
    RS_CUDA(cudaMalloc(&e->long_np, e->long_cap * 4));
    RS_CUDA(cudaMalloc(&e->long_ng, e->long_cap * 4));
    RS_CUDA(cudaMalloc(&e->n_long, 16));
    const size_t max_pieces = L / emb::kChunk + e->long_cap + 1;
    const size_t max_groups = L / (emb::kChunk * emb::kGroupPieces) + e->long_cap + 1;
    RS_CUDA(cudaMalloc(&e->ppart, max_pieces * e->dmax * 4));
    RS_CUDA(cudaMalloc(&e->pdesc, max_pieces * sizeof(uint4)));
    RS_CUDA(cudaMalloc(&e->gdesc, max_groups * sizeof(uint2)));
    RS_CUDA(cudaMalloc(&e->gpart, max_groups * e->dmax * 4));
    e->tiles_cap = L / kSortTile + T + 2;
    e->sort_scratch_bytes =
        std::max(radix_sort_scratch_bytes(L, T), radix_onesweep_scratch_bytes(L, e->tiles_cap)) + (4 << 20);
    RS_CUDA(cudaMalloc(&e->d_tiles, 3 * e->tiles_cap * 4));
    RS_CUDA(cudaMalloc(&e->sort_scratch, e->sort_scratch_bytes));
    // per-backward metadata: tpos[T+1] | wstart[T+1] | wtab[T] (class-major
    // window work map)
    const size_t meta = 3 * size_t(T) + 3;  // + the error word read back with tpos
    e->meta_words = meta;
    RS_CUDA(cudaMalloc(&e->d_meta, meta * 4));
    RS_CUDA(cudaHostAlloc(&e->h_meta, meta * 4, cudaHostAllocDefault));
    RS_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    delete e;
    throw;
  }
  return e;
}

// ------------------------------------------------------------------ slow-row staging
void emb_enable_cache(rs_emb* e, uint32_t nslots) {
  if (e->nslots) throw InvalidArgument("emb: the slow-row cache is already enabled");
  if (nslots == 0 || nslots >= emb::kClaim) throw InvalidArgument("emb: nslots out of range");
  cudaStream_t st = e->ctx->stream;
  uint64_t total_slow = 0;
  for (const auto& d : e->h_tables) total_slow += d.slow_rows;
  const uint64_t stride = e->rmax;  // bytes per slot / bounce row
  // one generation's rows fit in half the slots (nslots >= 2x a batch's rows)
  e->bcap = nslots / 2 + 1;
  const uint64_t bc = e->bcap;
  RS_CUDA(cudaMalloc(&e->staging, uint64_t(nslots) * stride));
  RS_CUDA(cudaMalloc(&e->slot_of, std::max<uint64_t>(total_slow, 1) * 4));
  RS_CUDA(cudaMalloc(&e->slot_gen, uint64_t(nslots) * 4));
  RS_CUDA(cudaMalloc(&e->slot_tab, uint64_t(nslots) * 4));
  RS_CUDA(cudaMalloc(&e->slot_row, uint64_t(nslots) * 4));
  RS_CUDA(cudaMalloc(&e->free_stack, uint64_t(nslots) * 4));
  // copy lists double-buffered by generation parity: with two batches staged
  // ahead, the claim for g+2 runs while g+1's lists may still be read
  RS_CUDA(cudaMalloc(&e->copy_list, 2 * bc * 4));
  RS_CUDA(cudaMalloc(&e->copy_tab, 2 * bc * 4));
  RS_CUDA(cudaMalloc(&e->copy_row, 2 * bc * 4));
  RS_CUDA(cudaMalloc(&e->wb_tab, bc * 4));
  RS_CUDA(cudaMalloc(&e->wb_row, bc * 4));
  RS_CUDA(cudaMalloc(&e->d_bin, bc * stride));
  RS_CUDA(cudaMalloc(&e->d_bout, bc * stride));
  RS_CUDA(cudaMalloc(&e->free_top, 4));
  RS_CUDA(cudaMalloc(&e->ncopy, 2 * 4));
  RS_CUDA(cudaMalloc(&e->n_wb, 4));
  RS_CUDA(cudaMalloc(&e->cache_err, 4));
  RS_CUDA(cudaHostAlloc(&e->h_bin, bc * stride, cudaHostAllocDefault));
  RS_CUDA(cudaHostAlloc(&e->h_bout, bc * stride, cudaHostAllocDefault));
  for (uint32_t** hp : {&e->h_ctab, &e->h_crow, &e->h_wtab, &e->h_wrow})
    RS_CUDA(cudaHostAlloc(hp, bc * 4, cudaHostAllocDefault));
  RS_CUDA(cudaHostAlloc(&e->h_cnt, 16, cudaHostAllocDefault));
  RS_CUDA(cudaMemsetAsync(e->slot_of, 0xFF, std::max<uint64_t>(total_slow, 1) * 4, st));
  RS_CUDA(cudaMemsetAsync(e->slot_gen, 0, uint64_t(nslots) * 4, st));
  RS_CUDA(cudaMemsetAsync(e->cache_err, 0, 4, st));
  std::vector<uint32_t> fs(nslots);
  std::iota(fs.begin(), fs.end(), 0u);
  RS_CUDA(cudaMemcpyAsync(e->free_stack, fs.data(), uint64_t(nslots) * 4, cudaMemcpyHostToDevice, st));
  const int top = int(nslots);
  RS_CUDA(cudaMemcpyAsync(e->free_top, &top, 4, cudaMemcpyHostToDevice, st));
  std::vector<TableDev> tc = e->h_tables;
  uint64_t base = 0;
  for (auto& d : tc) {
    d.slot_of = e->slot_of + base;
    d.staging = e->staging;
    d.stage_stride = stride;
    base += d.slow_rows;
  }
  RS_CUDA(cudaMalloc(&e->d_tables_c, sizeof(TableDev) * e->T));
  RS_CUDA(cudaMemcpyAsync(e->d_tables_c, tc.data(), sizeof(TableDev) * e->T, cudaMemcpyHostToDevice, st));
  {
    std::vector<uint32_t> st_list;
    for (uint32_t t = 0; t < e->T; ++t)
      if (e->h_tables[t].slow_rows) st_list.push_back(t);
    e->nslow_tabs = uint32_t(st_list.size());
    RS_CUDA(cudaMalloc(&e->d_slow_tabs, std::max<size_t>(1, st_list.size()) * 4));
    if (!st_list.empty())
      RS_CUDA(cudaMemcpyAsync(e->d_slow_tabs, st_list.data(), st_list.size() * 4, cudaMemcpyHostToDevice, st));
  }
  RS_CUDA(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
  RS_CUDA(cudaStreamCreateWithFlags(&e->side_out, cudaStreamNonBlocking));
  RS_CUDA(cudaStreamCreateWithFlags(&e->claim_stream, cudaStreamNonBlocking));
  for (cudaEvent_t* ev : {&e->ev_main, &e->ev_gather[0], &e->ev_gather[1], &e->ev_gather[2], &e->ev_gather[3],
                          &e->ev_claim[0], &e->ev_claim[1], &e->ev_claim[2], &e->ev_claim[3], &e->ev_evict[0],
                          &e->ev_evict[1], &e->ev_evict[2], &e->ev_evict[3]})
    RS_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
  RS_CUDA(cudaStreamSynchronize(st));
  // host threads: one gather pool (in) and one scatter pool (out), half of
  // the cores each, up to 16 / 8 (the two rarely run at once; with the
  // chunked write-back, 8 scatter threads on a 16-core box: RM1 step 3.65 ->
  // 3.47 ms over three same-box A/B runs vs 4)
  const unsigned hw = std::max(4u, std::thread::hardware_concurrency());
  auto env_threads = [](const char* name, unsigned dflt) {
    const char* v = getenv(name);
    const int n = v ? atoi(v) : 0;
    return n > 0 ? unsigned(n) : dflt;
  };
  e->pool = std::make_unique<rs::ThreadPool>(env_threads("RS_GATHER_THREADS", std::min(16u, hw / 2)));
  e->out_pool = std::make_unique<rs::ThreadPool>(env_threads("RS_SCATTER_THREADS", std::min(8u, hw / 2)));
  e->worker = std::make_unique<rs::TaskQueue>();
  e->out_worker = std::make_unique<rs::TaskQueue>();
  e->nslots = nslots;
}

static const char* kCacheErrMsg =
    "emb: slow-row cache out of slots; enable it with more slots "
    "(>= 4x the unique slow rows of a batch: up to four generations are live)";

// Reads and clears the device error word of the claim kernels.
static unsigned take_cache_error(rs_emb* e) {
  unsigned err = 0;
  RS_CUDA(cudaMemcpyAsync(&e->h_cnt[3], e->cache_err, 4, cudaMemcpyDeviceToHost, e->ctx->stream));
  RS_CUDA(cudaStreamSynchronize(e->ctx->stream));
  err = e->h_cnt[3];
  if (err) RS_CUDA(cudaMemsetAsync(e->cache_err, 0, 4, e->ctx->stream));
  return err;
}

// Host row of (table t, slow row r) in the pinned host tier.
static inline char* host_slow_row(rs_emb* e, uint32_t t, uint32_t r) {
  const TableDev& d = e->h_tables[t];
  return e->host_pool + (d.slow - e->host_pool_dev) + uint64_t(r) * d.rbytes;
}

// Worker task: rows claimed for generation g (claim event ev_claim[g & 3])
// host tier -> pinned bounce (CPU threads) -> HBM bounce (DMA) -> slots.
static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void stage_in_task(rs_emb* e, uint64_t g, uint64_t out_before) {
  static const bool dbg = getenv("RS_STAGE_DEBUG") != nullptr;
  const double t0 = dbg ? now_us() : 0;
  cudaStream_t s = e->side;
  // rows evicted by earlier generations must be in the host tier first
  if (out_before) e->out_worker->wait(out_before);
  RS_CUDA(cudaStreamSynchronize(s));  // the previous DMA out of h_bin is done
  RS_CUDA(cudaEventSynchronize(e->ev_claim[g & 3]));
  const double t1 = dbg ? now_us() : 0;
  const uint64_t cs = (g & 1) * e->bcap;  // this generation's copy-list set
  unsigned* ncopy = e->ncopy + (g & 1);
  RS_CUDA(cudaMemcpyAsync(e->h_cnt, ncopy, 4, cudaMemcpyDeviceToHost, s));
  RS_CUDA(cudaMemcpyAsync(e->h_cnt + 2, e->cache_err, 4, cudaMemcpyDeviceToHost, s));
  RS_CUDA(cudaStreamSynchronize(s));
  e->gen_err[g & 3] = e->h_cnt[2];  // read by begin_step before generation g runs
  const uint64_t n = std::min<uint64_t>(e->h_cnt[0], e->bcap);
  const uint64_t stride = e->rmax;
  if (n) {
    RS_CUDA(cudaMemcpyAsync(e->h_ctab, e->copy_tab + cs, n * 4, cudaMemcpyDeviceToHost, s));
    RS_CUDA(cudaMemcpyAsync(e->h_crow, e->copy_row + cs, n * 4, cudaMemcpyDeviceToHost, s));
    RS_CUDA(cudaStreamSynchronize(s));
    const double t2 = dbg ? now_us() : 0;
    // gather chunk c on the CPU while chunk c-1 is on the bus
    constexpr uint64_t kChunkRows = 16384;
    for (uint64_t c0 = 0; c0 < n; c0 += kChunkRows) {
      const uint64_t c1 = std::min(n, c0 + kChunkRows);
      e->pool->parallel_for(c1 - c0, [&](size_t b, size_t en) {
        for (size_t k = c0 + b; k < c0 + en; ++k) {
          const uint32_t t = e->h_ctab[k];
          memcpy(e->h_bin + k * stride, host_slow_row(e, t, e->h_crow[k]), e->h_tables[t].rbytes);
        }
      });
      RS_CUDA(cudaMemcpyAsync(e->d_bin + c0 * stride, e->h_bin + c0 * stride, (c1 - c0) * stride,
                              cudaMemcpyHostToDevice, s));
    }
    const double t3 = dbg ? now_us() : 0;
    if (dbg)
      fprintf(stderr, "stage_in g=%llu n=%llu t=%.0f wait=%.0fus lists=%.0fus gather+enqueue=%.0fus (%u threads)\n",
              (unsigned long long)g, (unsigned long long)n, t0, t1 - t0, t2 - t1, t3 - t2, e->pool->size());
    const unsigned grid = unsigned(std::min<uint64_t>((n + 7) / 8, uint64_t(sm_count()) * 4));
    emb::uvm_scatter_in_kernel<<<grid, 256, 0, s>>>(e->d_tables_c, e->copy_list + cs, e->copy_tab + cs, ncopy, e->bcap,
                                                   e->d_bin, e->staging, stride);
    RS_COUNT(1);
    RS_LAUNCH_CHECK();
  }
  RS_CUDA(cudaEventRecord(e->ev_gather[g & 3], s));
}

// Worker task: rows an eviction packed into d_bout (its event `evicted`)
// HBM bounce -> pinned bounce (DMA) -> host tier (CPU threads).
static void stage_out_task(rs_emb* e, cudaEvent_t evicted) {
  static const bool dbg = getenv("RS_STAGE_DEBUG") != nullptr;
  const double t0 = dbg ? now_us() : 0;
  cudaStream_t s = e->side_out;
  RS_CUDA(cudaEventSynchronize(evicted));
  const double t1 = dbg ? now_us() : 0;
  RS_CUDA(cudaMemcpyAsync(e->h_cnt + 1, e->n_wb, 4, cudaMemcpyDeviceToHost, s));
  RS_CUDA(cudaStreamSynchronize(s));
  const uint64_t n = std::min<uint64_t>(e->h_cnt[1], e->bcap);
  if (!n) return;
  const uint64_t stride = e->rmax;
  RS_CUDA(cudaMemcpyAsync(e->h_wtab, e->wb_tab, n * 4, cudaMemcpyDeviceToHost, s));
  RS_CUDA(cudaMemcpyAsync(e->h_wrow, e->wb_row, n * 4, cudaMemcpyDeviceToHost, s));
  // rows come back in chunks: the CPU scatters chunk c while chunk c+1 is on
  // the bus (the stage-out path was D2H then scatter, ~one step end to end)
  constexpr uint64_t kChunkRows = 16384;
  const uint64_t nch = (n + kChunkRows - 1) / kChunkRows;
  while (e->ev_out_chunk.size() < nch) {
    cudaEvent_t ev;
    RS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->ev_out_chunk.push_back(ev);
  }
  for (uint64_t c = 0; c < nch; ++c) {
    const uint64_t c0 = c * kChunkRows, c1 = std::min(n, c0 + kChunkRows);
    RS_CUDA(cudaMemcpyAsync(e->h_bout + c0 * stride, e->d_bout + c0 * stride, (c1 - c0) * stride,
                            cudaMemcpyDeviceToHost, s));
    RS_CUDA(cudaEventRecord(e->ev_out_chunk[c], s));
  }
  const double t2 = dbg ? now_us() : 0;
  for (uint64_t c = 0; c < nch; ++c) {
    const uint64_t c0 = c * kChunkRows, c1 = std::min(n, c0 + kChunkRows);
    RS_CUDA(cudaEventSynchronize(e->ev_out_chunk[c]));
    e->out_pool->parallel_for(c1 - c0, [&](size_t b, size_t en) {
      for (size_t k = c0 + b; k < c0 + en; ++k) {
        const uint32_t t = e->h_wtab[k];
        memcpy(host_slow_row(e, t, e->h_wrow[k]), e->h_bout + k * stride, e->h_tables[t].rbytes);
      }
    });
  }
  if (dbg)
    fprintf(stderr, "stage_out n=%llu t=%.0f wait_evict=%.0fus lists+enqueue=%.0fus d2h+scatter=%.0fus\n", (unsigned long long)n,
            t0, t1 - t0, t2 - t1, now_us() - t2);
}

// Evicts generation bit(s) `gen_bits` except rows of `keep` (caller's
// stream) and queues their return to the host tier.
static void evict(rs_emb* e, uint32_t gen_bits, uint32_t keep) {
  cudaStream_t st = e->ctx->stream;
  if (e->wb_seq) e->out_worker->wait(e->wb_seq);  // d_bout free again
  if (e->last_claim) RS_CUDA(cudaStreamWaitEvent(st, e->last_claim, 0));  // slot tables settled
  RS_CUDA(cudaMemsetAsync(e->n_wb, 0, 4, st));
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((e->nslots + 255) / 256, uint64_t(sm_count()) * 8)));
  emb::uvm_evict_kernel<<<grid, 256, 0, st>>>(e->d_tables_c, e->nslots, gen_bits, keep, e->slot_gen, e->slot_tab,
                                              e->slot_row, e->free_stack, e->free_top, e->staging, e->rmax,
                                              e->d_bout, e->wb_tab, e->wb_row, e->bcap, e->n_wb, e->cache_err);
  RS_COUNT(1);
  RS_LAUNCH_CHECK();
  // each eviction gets its own event: the host may run ahead and record the
  // next eviction before this task syncs (a shared event would then wait on
  // work queued behind a stream wait on this very pipeline)
  cudaEvent_t ev = e->ev_evict[e->n_evicts++ & 3];
  RS_CUDA(cudaEventRecord(ev, st));
  e->wb_seq = e->out_worker->post([e, ev] { stage_out_task(e, ev); });
}

// After the backward that used generation g: the generation finished one
// step EARLIER is evicted (its rows that neither g nor a pending prefetch
// needs go back to the host tier).  The one-step delay means a claim never
// needs a row whose write-back is still in flight: a claim for g+1 runs
// before g-1 is evicted (so it re-marks the still-staged row), and by the
// time g+2 is claimed, g-1's stage-out has had a whole step to finish.
static void enqueue_writeback(rs_emb* e, uint64_t g) {
  if (e->done_gen >= 0) {
    uint32_t keep = 1u << (g & 3);
    for (uint64_t p : e->pending) keep |= 1u << (p & 3);
    evict(e, 1u << (uint64_t(e->done_gen) & 3), keep);
  }
  e->done_gen = int64_t(g);
}

void emb_prefetch(rs_emb* e, uint64_t B, const uint32_t* off, const uint32_t* idx) {
  if (!e->nslots) throw InvalidArgument("emb_prefetch: enable the slow-row cache first");
  if (B == 0 || B > e->max_batch) throw InvalidArgument("emb_prefetch: batch outside [1, max_batch]");
  const uint64_t g = e->next_gen;
  // live generations: done (awaiting eviction), current, pending; g & 3 must be free
  const bool clash = e->pending.size() >= 2 ||
                     (e->done_gen >= 0 && (uint64_t(e->done_gen) & 3) == (g & 3)) ||
                     (e->cur_gen >= 0 && (uint64_t(e->cur_gen) & 3) == (g & 3));
  if (clash) throw InvalidArgument("emb_prefetch: at most two prefetched batches may be pending");
  ++e->next_gen;
  // claim (index + remap read per lookup, an atomic per new slow row) on the
  // side stream, after everything the caller queued so far (its inputs and
  // the last eviction) and before the next eviction (enqueue_writeback waits
  // for it): it overlaps the caller's next kernels
  RS_CUDA(cudaEventRecord(e->ev_main, e->ctx->stream));
  cudaStream_t st = e->claim_stream;
  RS_CUDA(cudaStreamWaitEvent(st, e->ev_main, 0));
  const uint64_t cs = (g & 1) * e->bcap;
  RS_CUDA(cudaMemsetAsync(e->ncopy + (g & 1), 0, 4, st));
  if (e->nslow_tabs) {
    const uint64_t work = uint64_t(e->nslow_tabs) * ((B + 31) / 32);
    emb::uvm_claim_kernel<<<unsigned(std::max<uint64_t>(1, std::min<uint64_t>((work + 7) / 8, uint64_t(sm_count()) * 8))),
                            256, 0, st>>>(
        e->d_tables_c, e->d_slow_tabs, e->nslow_tabs, B, off, idx, 1u << (g & 3), e->slot_gen,
        e->slot_tab, e->slot_row, e->free_stack, e->free_top, e->copy_list + cs, e->copy_tab + cs,
        e->copy_row + cs, e->bcap, e->ncopy + (g & 1), e->cache_err);
    RS_COUNT(1);
    RS_LAUNCH_CHECK();
  }
  RS_CUDA(cudaEventRecord(e->ev_claim[g & 3], st));
  e->last_claim = e->ev_claim[g & 3];
  const uint64_t ob = e->out_worker->posted();
  e->gather_seq[g & 3] = e->worker->post([e, g, ob] { stage_in_task(e, g, ob); });
  e->pending.push_back(g);
  e->staged_dirty = true;
}

// Writes every staged row back and drops pending prefetches (they would
// refetch); afterwards the host tier is authoritative again.
void emb_flush(rs_emb* e) {
  if (!e->nslots || !e->staged_dirty) return;
  e->worker->drain();
  for (cudaEvent_t ev : e->ev_gather) RS_CUDA(cudaStreamWaitEvent(e->ctx->stream, ev, 0));
  // a generation's rows fit the bounce buffers: evict one generation at a time
  for (uint32_t b = 0; b < 4; ++b) evict(e, 1u << b, 0u);
  e->out_worker->drain();
  e->done_gen = -1;
  RS_CUDA(cudaStreamSynchronize(e->ctx->stream));
  e->pending.clear();
  e->cur_gen = -1;
  e->staged_dirty = false;
  for (unsigned& x : e->gen_err) x = 0;
  // the cache is empty and consistent again; a failed claim is still reported
  if (take_cache_error(e)) throw InvalidArgument(kCacheErrMsg);
}

// Picks the tables for a forward: the oldest prefetched batch (staged rows)
// or, without a prefetch, the zero-copy path.
static void begin_step(rs_emb* e) {
  if (e->cur_gen >= 0) {  // previous staged forward without a backward
    const uint64_t g = uint64_t(e->cur_gen);
    e->cur_gen = -1;
    enqueue_writeback(e, g);
  }
  if (!e->pending.empty()) {
    const uint64_t g = e->pending.front();
    e->pending.erase(e->pending.begin());
    e->cur_gen = int64_t(g);
    e->worker->wait(e->gather_seq[g & 3]);  // its copies are enqueued
    if (e->gen_err[g & 3]) {
      // some of this batch's slow rows got no slot: refuse to run it (a later
      // staged batch could otherwise re-read a row this one updates in the
      // host tier); flush() empties the cache and clears the error
      e->cur_gen = -1;
      e->pending.insert(e->pending.begin(), g);
      throw InvalidArgument(kCacheErrMsg);
    }
    RS_CUDA(cudaStreamWaitEvent(e->ctx->stream, e->ev_gather[g & 3], 0));
    e->cur_tables = e->d_tables_c;
  } else {
    emb_flush(e);
    e->cur_tables = e->d_tables;
  }
}

void emb_init_weights(rs_emb* e, uint64_t seed, float scale) {
  emb_flush(e);
  cudaStream_t st = e->ctx->stream;
  for (uint32_t t = 0; t < e->T; ++t) {
    const TableDev& d = e->h_tables[t];
    const uint64_t n = d.hash_size * (d.dim / 4);
    unsigned g = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(sm_count()) * 16));
    emb::init_kernel<<<std::max(1u, g), 256, 0, st>>>(d, e->table_ids[t], seed, scale);
  }
  RS_LAUNCH_CHECK();
}

static uint32_t fwd_chunk() {
  static const uint32_t c = [] {
    const char* v = getenv("RS_FWD_CHUNK");
    return v ? uint32_t(std::max(1, atoi(v))) : 4u;
  }();
  return c;
}

// wide rows (VPL > 1) the same way: B200 RM3-like (dim 256 fp16, G 32, VPL 2):
// (2 rows, 4 CTAs/SM) 5.96 ms, (2, 6) 5.98, (4, 4) 6.71, (4, 2) 7.27, (8, 1) 10.18
template <int G, int VPL, class E, int UNR_ = 2, int MINB_ = (VPL == 1 ? 8 : VPL == 2 ? 4 : VPL == 4 ? 3 : 2)>
static void launch_fwd(rs_emb* e, const rs_emb::Class& c, uint64_t B, const uint32_t* off,
                       const uint32_t* idx, const OutMap& out, uint64_t stride, unsigned long long* hits,
                       cudaStream_t st) {
  constexpr int BPW = 32 / G;
  const uint64_t warps = (B + BPW - 1) / BPW * c.tables.size();  // bag-groups
  // persistent: one full wave; the class's own chunk counter (classes run
  // on two streams)
  uint32_t* work = e->d_work + (&c - e->classes.data());
  const uint32_t chunk = fwd_chunk();
  const uint64_t chunks = (warps + chunk - 1) / chunk;
  if (warps >= (uint64_t(1) << 32)) throw InvalidArgument("emb_forward: batch too large for one launch");
  // (rows in flight per group, CTAs/SM), B200 RM1 all-HBM (op_bench, one box,
  // two runs): (2, 8) 1.26-1.31 ms, (2, 6) 1.29-1.30, (3, 6) 1.35, (4, 6)
  // 1.39-1.40, (4, 5) 1.41-1.42 — with the chunked schedule, occupancy wins
  // over rows in flight per group (the 32-register cap spills only in the
  // per-bag cursor code)
  constexpr int MINB = MINB_;
  const bool fk = e->resolved;  // keys resolved by resolve_kernel: the gather reads slot keys
  auto kern = fk ? (c.full ? emb::forward_kernel<G, VPL, UNR_, MINB, E, true, true>
                           : emb::forward_kernel<G, VPL, UNR_, MINB, E, false, true>)
                 : (c.full ? emb::forward_kernel<G, VPL, UNR_, MINB, E, true, false>
                           : emb::forward_kernel<G, VPL, UNR_, MINB, E, false, false>);
  if (fk) idx = e->keys;
  static const int per_sm = [&] {
    int n = 0;
    RS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, emb::forward_kernel<G, VPL, UNR_, MINB, E, false>,
                                                          emb::kFwdThreads, 0));
    return std::max(1, n);
  }();
  const unsigned grid = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>(uint64_t(sm_count()) * per_sm, (chunks * 32 + emb::kFwdThreads - 1) / emb::kFwdThreads)));
  RS_CUDA(cudaMemsetAsync(work, 0, 4, st));
  kern<<<grid, emb::kFwdThreads, 0, st>>>(
      e->cur_tables, c.d_list, uint32_t(c.tables.size()), uint32_t(B), off, idx, out, stride, hits, e->d_unbacked,
      e->keys, e->vals, uint64_t(e->max_lookups), e->d_err, work, chunk);
  RS_COUNT(1);
}

// One launch per lane class, instantiated per (G, VPL) and storage type.
template <class E>
static void launch_fwd_class(rs_emb* e, const rs_emb::Class& c, uint64_t B, const uint32_t* off,
                             const uint32_t* idx, const OutMap& om, uint64_t stride, unsigned long long* h,
                             cudaStream_t st) {
  switch (c.G * 100 + c.VPL) {
    case 101: launch_fwd<1, 1, E>(e, c, B, off, idx, om, stride, h, st); break;
    case 201: launch_fwd<2, 1, E>(e, c, B, off, idx, om, stride, h, st); break;
    case 401: launch_fwd<4, 1, E>(e, c, B, off, idx, om, stride, h, st); break;
    case 801: launch_fwd<8, 1, E>(e, c, B, off, idx, om, stride, h, st); break;
    case 1601: launch_fwd<16, 1, E>(e, c, B, off, idx, om, stride, h, st); break;
    case 3201: launch_fwd<32, 1, E>(e, c, B, off, idx, om, stride, h, st); break;
    case 3202: launch_fwd<32, 2, E>(e, c, B, off, idx, om, stride, h, st); break;
    case 3204: launch_fwd<32, 4, E>(e, c, B, off, idx, om, stride, h, st); break;
    case 3208: launch_fwd<32, 8, E>(e, c, B, off, idx, om, stride, h, st); break;
    default: throw Error(-9, "emb_forward: unsupported lane class");
  }
}

void emb_forward(rs_emb* e, uint64_t B, const uint32_t* off, const uint32_t* idx, float* out,
                 uint64_t* hits) {
  OutMap om{};
  om.out0 = out;
  om.bl = B;
  om.n = 1;
  emb_forward_map(e, B, off, idx, om, e->total_dim, hits);
}

void emb_forward_map(rs_emb* e, uint64_t B, const uint32_t* off, const uint32_t* idx, const OutMap& om,
                     uint64_t stride, uint64_t* hits) {
  if (B == 0 || B > e->max_batch) throw InvalidArgument("emb_forward: batch outside [1, max_batch]");
  begin_step(e);
  e->t_fwd.begin(e->ctx->stream);
  e->keys_off = off;
  e->keys_idx = idx;
  e->keys_B = B;
  auto* h = reinterpret_cast<unsigned long long*>(hits);
  // lane classes write disjoint columns, keys and hit counters: every other
  // class runs on a forked stream so one launch's tail overlaps the next
  cudaStream_t main = e->ctx->stream;
  // index resolution as its own streaming pass, then the gather from slot
  // keys (B200 RM1: forward 1.22 -> 1.07 ms incl. the pass, same-box A/B);
  // RS_FWD_RESOLVE=0 resolves inside the gather and writes the keys there
  static const bool resolve = [] {
    const char* v = getenv("RS_FWD_RESOLVE");
    return !(v && v[0] == '0');
  }();
  e->resolved = resolve && e->keys;
  if (e->resolved) {
    const uint64_t nb = uint64_t(e->T) * B;
    const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((nb / 32 + 7) / 8, uint64_t(sm_count()) * 16)));
    emb::resolve_kernel<<<g, 256, 0, main>>>(e->cur_tables, e->T, uint32_t(B), off, idx, e->keys, e->vals,
                                             uint64_t(e->max_lookups), e->d_err);
    RS_COUNT(1);
  }
  const bool fork = e->classes.size() > 1;
  if (fork) {
    RS_CUDA(cudaEventRecord(e->ev_fork, main));
    RS_CUDA(cudaStreamWaitEvent(e->fwd_side, e->ev_fork, 0));
  }
  for (size_t ci = 0; ci < e->classes.size(); ++ci) {
    const auto& c = e->classes[ci];
    cudaStream_t st = (ci & 1) ? e->fwd_side : main;
    if (c.EB == 2) launch_fwd_class<__half>(e, c, B, off, idx, om, stride, h, st);
    else launch_fwd_class<float>(e, c, B, off, idx, om, stride, h, st);
  }
  if (fork) {
    RS_CUDA(cudaEventRecord(e->ev_join, e->fwd_side));
    RS_CUDA(cudaStreamWaitEvent(main, e->ev_join, 0));
  }
  RS_LAUNCH_CHECK();
  e->t_fwd.end(e->ctx->stream);
}

void emb_kernel_times(rs_emb* e, double* fwd_ms, uint64_t* n_fwd, double* bwd_ms, uint64_t* n_bwd, int reset) {
  e->t_fwd.harvest();
  e->t_bwd.harvest();
  if (fwd_ms) *fwd_ms = e->t_fwd.ms;
  if (n_fwd) *n_fwd = e->t_fwd.count;
  if (bwd_ms) *bwd_ms = e->t_bwd.ms;
  if (n_bwd) *n_bwd = e->t_bwd.count;
  if (reset) {
    e->t_fwd.ms = e->t_bwd.ms = 0;
    e->t_fwd.count = e->t_bwd.count = 0;
  }
}

#ifndef RS_SEG_MINB
#define RS_SEG_MINB 4
#endif
// Short-segment bag pass for one lane class over its window range [wlo, whi).
template <int G, int VPL, int UNR, int MINB, class E>
static void launch_segs_v(rs_emb* e, const emb::BwdArgs& a, uint32_t ci, uint64_t max_windows, cudaStream_t st) {
  // the class's window range is on the device (bwd_plan_kernel): persistent
  // grid, capped by the class's largest possible window count
  const uint64_t est = max_windows * 8 / (uint64_t(emb::kBwdWarps) * (32 / G)) + 1;
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(est, uint64_t(sm_count()) * MINB)));
  emb::bwd_seg_kernel<G, VPL, UNR, MINB, E><<<grid, emb::kBwdThreads, 0, st>>>(
      a, e->segs, e->sbase, e->d_cw, ci, e->longs, e->long_np, e->long_ng, e->n_long);
  RS_COUNT(1);
}

template <int G, int VPL, class E>
static void launch_segs(rs_emb* e, const emb::BwdArgs& a, uint32_t ci, uint64_t max_windows, cudaStream_t st) {
  if constexpr (VPL == 1) launch_segs_v<G, 1, 4, RS_SEG_MINB, E>(e, a, ci, max_windows, st);
  // wide rows: B200 RM3-like (dim 256 fp16): (2 rows, 4 CTAs/SM) 16.9-17.0 ms
  // backward, (1, 4) 16.9-17.0, (1, 3) 17.0, (2, 3) 17.3, (2, 2) 18.5
  else launch_segs_v<G, VPL, 2, (VPL >= 8 ? 2 : 4), E>(e, a, ci, max_windows, st);
}

template <class E>
static void launch_segs_class(rs_emb* e, const rs_emb::Class& c, const emb::BwdArgs& a, uint32_t ci, uint64_t mw,
                              cudaStream_t cs) {
  switch (c.G * 100 + c.VPL) {
    case 101: launch_segs<1, 1, E>(e, a, ci, mw, cs); break;
    case 201: launch_segs<2, 1, E>(e, a, ci, mw, cs); break;
    case 401: launch_segs<4, 1, E>(e, a, ci, mw, cs); break;
    case 801: launch_segs<8, 1, E>(e, a, ci, mw, cs); break;
    case 1601: launch_segs<16, 1, E>(e, a, ci, mw, cs); break;
    case 3201: launch_segs<32, 1, E>(e, a, ci, mw, cs); break;
    case 3202: launch_segs<32, 2, E>(e, a, ci, mw, cs); break;
    case 3204: launch_segs<32, 4, E>(e, a, ci, mw, cs); break;
    case 3208: launch_segs<32, 8, E>(e, a, ci, mw, cs); break;
    default: throw Error(-9, "emb_backward: unsupported lane class");
  }
}

// Long segments: groups of 64 pieces, then one warp per segment (full warps,
// VPL of the widest table).
template <int VPL>
static void launch_long(rs_emb* e, const emb::BwdArgs& a) {
  const unsigned g = unsigned(sm_count()) * 8;
  cudaStream_t st = e->ctx->stream;
  emb::bwd_piece_desc_kernel<<<g, emb::kBwdThreads, 0, st>>>(e->longs, e->n_long, e->long_np, e->long_ng, e->pdesc,
                                                             e->gdesc);
  emb::bwd_lpiece_kernel<16, 2 * VPL><<<g, emb::kBwdThreads, 0, st>>>(a, e->pdesc, e->n_long, e->ppart);
  emb::bwd_group_kernel<VPL><<<g, emb::kBwdThreads, 0, st>>>(a, e->longs, e->n_long, e->long_np, e->gdesc,
                                                             e->ppart, e->gpart);
  emb::bwd_long_kernel<VPL><<<g, emb::kBwdThreads, 0, st>>>(a, e->longs, e->n_long, e->long_ng, e->gpart);
  RS_COUNT(4);
}

void emb_backward(rs_emb* e, uint64_t B, const uint32_t* off, const uint32_t* idx, const float* grad,
                  float lr) {
  if (B == 0 || B > e->max_batch) throw InvalidArgument("emb_backward: batch outside [1, max_batch]");
  // a backward belongs to the last forward's batch: staged rows if that batch
  // was prefetched, else the zero-copy path
  if (e->cur_gen < 0) {
    emb_flush(e);
    e->cur_tables = e->d_tables;
  }
  struct Release {
    rs_emb* e;
    ~Release() {
      if (e->cur_gen >= 0) {
        const uint64_t g = uint64_t(e->cur_gen);
        e->cur_gen = -1;
        try {
          enqueue_writeback(e, g);
        } catch (...) {
        }
      }
    }
  } release{e};
  cudaStream_t st = e->ctx->stream;
  const uint32_t T = e->T;
  uint32_t* herr = e->h_meta + e->meta_words - 1;
  // keys from the forward of this very batch?  (the sort below consumes them)
  const bool have_keys = e->keys_off == off && e->keys_idx == idx && e->keys_B == B;
  e->keys_off = nullptr;
  // Everything is enqueued before the host looks at anything: the plan
  // (validation, work map, sort tiles) is computed on the device from the
  // offsets, so the GPU runs the backward straight after the forward.  The
  // host then waits only for the plan's error word and raises afterwards
  // (an empty plan makes every later kernel a no-op).
  e->t_bwd.begin(st);
  uint32_t* d_tpos = e->d_meta;
  uint32_t* d_wstart = e->d_meta + T + 1;
  uint32_t* d_wtab = e->d_meta + 2 * (T + 1);
  const uint32_t tcap = uint32_t(e->tiles_cap);
  {
    emb::BwdPlan pl{off, B, T, e->d_order, e->d_cpos, uint32_t(e->classes.size()), e->max_lookups,
                    d_tpos, d_wstart, d_wtab, e->d_cw, e->d_tiles, tcap, e->d_nt, e->d_err};
    emb::bwd_plan_kernel<<<1, 1024, 0, st>>>(pl);
    RS_COUNT(1);
    if (!have_keys) {  // a batch the last forward did not see: keys from the (validated) offsets
      const uint64_t nb = uint64_t(e->T) * B;
      unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((nb / 32 + 7) / 8, uint64_t(sm_count()) * 16)));
      emb::keygen_kernel<<<g, 256, 0, st>>>(e->d_tables, e->T, B, off, idx, e->keys, e->vals, e->d_err);
      emb::bwd_plan_gate_kernel<<<1, 256, 0, st>>>(pl);  // an index error empties the plan too
      RS_COUNT(2);
    }
    RS_CUDA(cudaMemcpyAsync(herr, e->d_err, 4, cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaEventRecord(e->ev_err, st));
  }
  const uint64_t Lmax = e->max_lookups;
  Scratch scr;
  scr.base = e->sort_scratch;
  scr.cap = e->sort_scratch_bytes;
  uint32_t* skeys = e->keys;
  uint32_t* svals = e->vals;
  {
    // segmented sort: each table's CSR range sorted on its own (slot keys)
    TileMap tm;
    tm.pos = e->d_tiles;
    tm.cidx = e->d_tiles + tcap;
    tm.cstride = e->d_tiles + 2 * size_t(tcap);
    tm.ntd = e->d_nt;
    // one kernel per pass with decoupled look-back (B200 RM1: backward 2.07 ->
    // 1.99 ms, three A/B runs); RS_SORT_ONESWEEP=0 selects the upsweep /
    // count-scan / downsweep passes
    static const bool onesweep = [] {
      const char* v = getenv("RS_SORT_ONESWEEP");
      return !(v && v[0] == '0');
    }();
    if (onesweep)
      radix_sort_pairs_onesweep(e->keys, e->vals, Lmax, int(e->key_bits), scr, st, tm, tcap - 1, &skeys, &svals);
    else
      radix_sort_pairs(e->keys, e->vals, Lmax, int(e->key_bits), scr, st, tm, tcap - 1, &skeys, &svals);
  }
  emb::BwdArgs a{e->cur_tables, T, d_tpos, skeys, svals, grad, e->total_dim, e->dmax, lr, e->eps, e->opt};
  // segment list: count heads per window, scan, write descriptors
  const uint64_t Wmax = (Lmax + emb::kChunk - 1) / emb::kChunk + T;
  emb::WorkMap wm{d_wstart, d_wtab, T};
  const unsigned gs = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((Wmax + 7) / 8, uint64_t(sm_count()) * 16)));
  emb::bwd_seg_scan_kernel<false><<<gs, 256, 0, st>>>(a, wm, e->scount, nullptr, nullptr);
  exclusive_scan<uint32_t>(ArrayIn<uint32_t>{e->scount}, Wmax, e->sbase, e->sbase + Wmax, scr, st);
  emb::bwd_seg_scan_kernel<true><<<gs, 256, 0, st>>>(a, wm, nullptr, e->sbase, e->segs);
  RS_COUNT(2);
  // gradients arriving from other ranks (exchange.cu) are read from here on;
  // the plan, sort and segment list above overlapped their transfer
  if (e->grad_ready) {
    RS_CUDA(cudaStreamWaitEvent(st, e->grad_ready, 0));
    e->grad_ready = nullptr;
  }
  // short segments per lane class (long ones are listed)
  RS_CUDA(cudaMemsetAsync(e->n_long, 0, 16, st));
  // classes update disjoint rows (the long list is an atomic append): every
  // other class on the forked stream, as in the forward
  const bool fork = e->classes.size() > 1;
  if (fork) {
    RS_CUDA(cudaEventRecord(e->ev_fork, st));
    RS_CUDA(cudaStreamWaitEvent(e->fwd_side, e->ev_fork, 0));
  }
  for (size_t ci = 0; ci < e->classes.size(); ++ci) {
    const auto& c = e->classes[ci];
    const uint64_t mw = Wmax;
    cudaStream_t cs = (ci & 1) ? e->fwd_side : st;
    if (c.EB == 2) launch_segs_class<__half>(e, c, a, uint32_t(ci), mw, cs);
    else launch_segs_class<float>(e, c, a, uint32_t(ci), mw, cs);
  }
  if (fork) {
    RS_CUDA(cudaEventRecord(e->ev_join, e->fwd_side));
    RS_CUDA(cudaStreamWaitEvent(st, e->ev_join, 0));
  }
  // long segments: piece / group descriptors, piece sums, group sums, final sums + updates
  switch (e->bwd_vpl) {
    case 1: launch_long<1>(e, a); break;
    case 2: launch_long<2>(e, a); break;
    case 4: launch_long<4>(e, a); break;
    case 8: launch_long<8>(e, a); break;
    default: throw Error(-9, "emb_backward: unsupported dim");
  }
  e->t_bwd.end(st);
  RS_LAUNCH_CHECK();
  // the plan's verdict (the GPU is already past it or running the backward)
  RS_CUDA(cudaEventSynchronize(e->ev_err));
  if (const unsigned bad = *herr) {
    RS_CUDA(cudaMemsetAsync(e->d_err, 0, 4, st));
    // the offsets first (an index read through bad offsets is meaningless)
    if (bad & 4u) throw InvalidArgument("emb_backward: offsets must start at 0");
    if (bad & 8u) throw InvalidArgument("emb_backward: more lookups than max_lookups");
    if (bad & 16u) throw InvalidArgument("emb_backward: offsets must be non-decreasing");
    if (bad & 2u) throw InvalidArgument("emb: more lookups than max_lookups");
    throw InvalidArgument("emb: an index is outside its table's hash_size");
  }
}

void emb_read_rows(rs_emb* e, uint32_t t, const uint32_t* rows, uint64_t n, float* out, float* mom) {
  if (t >= e->T) throw InvalidArgument("emb_read_rows: table index out of range");
  if (e->cur_gen >= 0) {  // a staged forward without its backward yet
    const uint64_t g = uint64_t(e->cur_gen);
    e->cur_gen = -1;
    enqueue_writeback(e, g);
  }
  emb_flush(e);
  cudaStream_t st = e->ctx->stream;
  const TableDev& d = e->h_tables[t];
  for (uint64_t i = 0; i < n; ++i)
    if (rows[i] >= d.hash_size) throw InvalidArgument("emb_read_rows: row out of range");
  if (n == 0) return;
  Scratch scr = e->ctx->scratch(n * (4 + 4 + size_t(d.dim) * 4) + (1 << 20));
  uint32_t* d_rows = stage(rows, n, false, scr, st);
  float* d_out = scr.take<float>(n * d.dim);
  float* d_mom = scr.take<float>(n);
  unsigned g = unsigned(std::min<uint64_t>((n * d.dim / 4 + 255) / 256, uint64_t(sm_count()) * 8));
  emb::read_rows_kernel<<<std::max(1u, g), 256, 0, st>>>(d, d_rows, n, d_out, d_mom);
  RS_LAUNCH_CHECK();
  RS_CUDA(cudaMemcpyAsync(out, d_out, n * d.dim * 4, cudaMemcpyDeviceToHost, st));
  if (mom) RS_CUDA(cudaMemcpyAsync(mom, d_mom, n * 4, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
}

void emb_free(rs_emb* e) {
  if (e) cudaStreamSynchronize(e->ctx->stream);
  delete e;
}

void emb_unbacked(rs_emb* e, uint64_t* lookups, uint64_t* rows, int reset) {
  cudaStream_t st = e->ctx->stream;
  if (lookups) {
    RS_CUDA(cudaMemcpyAsync(lookups, e->d_unbacked, 8 * size_t(e->T), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
  }
  if (reset) RS_CUDA(cudaMemsetAsync(e->d_unbacked, 0, 8 * size_t(e->T), st));
  if (rows) std::copy(e->unbacked_rows.begin(), e->unbacked_rows.end(), rows);
}

void emb_memory(const rs_emb* e, uint64_t* hbm, uint64_t* host) {
  if (hbm) *hbm = e->fast_bytes + e->remap_bytes;
  if (host) *host = e->host_bytes;
}

uint32_t emb_num_tables(const rs_emb* e) { return e->T; }
uint32_t emb_table_id(const rs_emb* e, uint32_t t) { return e->table_ids.at(t); }
uint32_t emb_table_dim(const rs_emb* e, uint32_t t) { return e->h_tables.at(t).dim; }
rs_context* emb_context(const rs_emb* e) { return e->ctx; }
void emb_set_grad_ready(rs_emb* e, cudaEvent_t ev) { e->grad_ready = ev; }

}  // namespace rs
