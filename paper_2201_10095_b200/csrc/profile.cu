// HP1 — the training-data profiler on the GPU.
//
//   K0 hash_ids      raw u64 -> mix64(raw) % H           inc/workload.hpp:28-31
//   K1 hash_hist     per-sample selection + per-row histogram
//                                                        core/src/profiler.cpp:68-112
//   K2 rank          compact accessed rows -> stable radix sort on (table,
//                    count desc) over row-ascending input -> u64 prefix ->
//                    access_cdf + 101-step ICDF          core/src/profiler.cpp:114-159
//
// Bit-exactness: every count is an exact integer; access_cdf is the IEEE
// division double(cum)/double(total) of exact u64s (correctly rounded on both
// CPU and GPU); the ICDF uses the reference's integer test
// 100*prefix(k) >= i*total (core/src/profiler.cpp:38).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>

#include "../../include/shardplan_gpu.h"
#include "context.cuh"

struct rs_profile {
  uint32_t J = 0;
  uint64_t selected = 0;
  std::vector<uint32_t> table_ids;
  std::vector<double> coverage, avg_pooling;
  std::vector<uint64_t> distinct, total, present;
  std::vector<uint64_t> icdf;   // J * 101
  std::vector<uint64_t> start;  // J + 1 offsets into rows / cdf
  // rows_by_rank / access_cdf of all tables: pinned host copies (D2H straight
  // from the rank kernels) and the device ranking (feeds build_remap)
  // (pinned blocks come from / return to the context's pool; the device
  // ranking is stream-ordered memory, so neither allocation nor release
  // synchronises the device)
  size_t nd = 0;
  uint32_t* rows = nullptr;
  double* cdf = nullptr;
  uint32_t* d_rows = nullptr;
  size_t rows_cap = 0, cdf_cap = 0;
  std::shared_ptr<rs::PinnedPool> pool;
  cudaStream_t stream = nullptr;
  ~rs_profile() {
    if (d_rows) cudaFreeAsync(d_rows, stream);
    if (pool) {
      pool->give(rows, rows_cap);
      pool->give(cdf, cdf_cap);
    }
  }
  // grows the three arrays to hold n more entries (groups append in order)
  void grow(size_t n, cudaStream_t st) {
    const size_t m = std::max<size_t>(nd + n, 1);
    size_t rc = 0, cc = 0;
    auto* r2 = static_cast<uint32_t*>(pool->take(m * 4, &rc));
    auto* c2 = static_cast<double*>(pool->take(m * 8, &cc));
    uint32_t* d2 = nullptr;
    RS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d2), m * 4, st));
    if (nd) {
      RS_CUDA(cudaStreamSynchronize(st));
      memcpy(r2, rows, nd * 4);
      memcpy(c2, cdf, nd * 8);
      RS_CUDA(cudaMemcpyAsync(d2, d_rows, nd * 4, cudaMemcpyDeviceToDevice, st));
    }
    if (d_rows) RS_CUDA(cudaFreeAsync(d_rows, st));
    pool->give(rows, rows_cap);
    pool->give(cdf, cdf_cap);
    rows = r2;
    cdf = c2;
    d_rows = d2;
    rows_cap = rc;
    cdf_cap = cc;
  }
};

namespace rs {
namespace prof {

constexpr uint64_t kProfileStream = 0x70726f66ULL;  // "prof", profiler.cpp:29
constexpr int kHistThreads = 256;
constexpr uint32_t kMaxSmemTables = 4096;
constexpr unsigned kErrUnknownTable = 1u;
constexpr unsigned kErrRowRange = 2u;

__device__ __forceinline__ int lookup_table(const uint32_t* __restrict__ sorted_ids,
                                            const uint32_t* __restrict__ sorted_idx,
                                            uint32_t J, uint32_t id) {
  uint32_t lo = 0, hi = J;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (sorted_ids[mid] < id) lo = mid + 1;
    else hi = mid;
  }
  return (lo < J && sorted_ids[lo] == id) ? int(sorted_idx[lo]) : -1;
}

__device__ __forceinline__ bool sample_selected(uint64_t s, double rate, uint64_t seed) {
  return rate >= 1.0 || first_double(derive_stream(seed, s, kProfileStream)) < rate;
}

// |{s < S : selected(s)}| — the coverage denominator (profiler.cpp:68-74).
__global__ void count_selected(uint64_t S, double rate, uint64_t seed,
                               unsigned long long* out) {
  uint64_t c = 0;
  for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < S;
       s += uint64_t(gridDim.x) * blockDim.x)
    c += sample_selected(s, rate, seed);
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

struct Tables {
  const uint32_t* sorted_ids;
  const uint32_t* sorted_idx;
  const uint64_t* base;   // counter offset of table index t (group-local)
  const uint64_t* hsize;
  const uint64_t* magic;
  uint32_t J;
  uint32_t t_lo, t_hi;    // table-index range counted by this launch
};

// K1.  Each warp takes 32 records (sample selection, table lookup, length),
// scans their lengths, and expands them into a shared-memory map of the
// warp's flattened id stream: for every id its table and its position in the
// ids array (32 lanes write one record at a time, so any length mix costs
// ~2 stores per 32 ids).  The ids are then processed 32 at a time with
// coalesced loads and no per-id record search.
//
// Zipf heads: same-address atomics serialise in the L2 atomic unit
// (B300_MICROARCH.md: "LTS atomic-ALU serializes per-address"), so one hot
// row hammered from every SM bounds the whole pass.  Large calls therefore
// run in two phases: a sample of the records (1/64) is counted straight into
// the global counters; rows whose sample count reaches a threshold form the
// HOT set (at most kHotMax rows — the Zipf head); the rest of the records run
// with the hot set in a per-CTA shared-memory hash (read-only keys, no CAS)
// whose counters take the hot increments, flushed once per CTA at the end.
// Other rows are counted with global atomics (no contention: the tail is
// spread).  Integer adds commute, so counts are exact and order-independent.
constexpr int kHotSlots = 8192;  // power of two
constexpr int kHotMax = kHotSlots / 2;
constexpr uint32_t kHotEmpty = 0xFFFFFFFFu;
constexpr int kWin = 256;         // ids per warp window of the expansion map
constexpr int kHistWarps = kHistThreads / 32;

__device__ __forceinline__ uint32_t hot_hash(uint32_t addr) { return (addr * 2654435761u) >> 19; }

template <bool RAW, bool HOT>
__global__ void __launch_bounds__(kHistThreads)
hash_hist(const uint64_t* __restrict__ rec_sample, const uint32_t* __restrict__ rec_table,
          const uint64_t* __restrict__ rec_offset, const uint32_t* __restrict__ rec_len,
          uint64_t r_lo, uint64_t r_hi, const uint32_t* __restrict__ ids,
          const uint64_t* __restrict__ raw, Tables tp, double rate, uint64_t seed,
          bool count_records, const uint32_t* __restrict__ hot_list,
          const unsigned* __restrict__ n_hot, uint32_t* __restrict__ counters,
          unsigned long long* __restrict__ present, unsigned long long* __restrict__ accesses,
          unsigned* __restrict__ err) {
  extern __shared__ uint32_t sm[];
  uint32_t* hkeys = sm;
  uint32_t* hvals = sm + (HOT ? kHotSlots : 0);
  uint32_t* mtab = sm + (HOT ? 2 * kHotSlots : 0);       // [warps][kWin] table index
  uint32_t* msrc = mtab + kHistWarps * kWin;              // [warps][kWin] ids position
  const bool use_sm = count_records && tp.J <= kMaxSmemTables;
  uint32_t* pres_s = msrc + kHistWarps * kWin;
  uint32_t* acc_s = pres_s + (use_sm ? tp.J : 0);
  if (HOT) {
    for (uint32_t i = threadIdx.x; i < kHotSlots; i += blockDim.x) {
      hkeys[i] = kHotEmpty;
      hvals[i] = 0;
    }
  }
  if (use_sm)
    for (uint32_t i = threadIdx.x; i < 2 * tp.J; i += blockDim.x) pres_s[i] = 0;
  __syncthreads();
  if (HOT) {
    const uint32_t nh = min(*n_hot, uint32_t(kHotMax));
    for (uint32_t i = threadIdx.x; i < nh; i += blockDim.x) {
      const uint32_t a = hot_list[i];
      uint32_t h = hot_hash(a);
      while (atomicCAS(&hkeys[h], kHotEmpty, a) != kHotEmpty) h = (h + 1) & (kHotSlots - 1);
    }
    __syncthreads();
  }

  const int lane = threadIdx.x & 31;
  uint32_t* wtab = mtab + (threadIdx.x >> 5) * kWin;
  uint32_t* wsrc = msrc + (threadIdx.x >> 5) * kWin;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t c = r_lo / 32 + ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); c * 32 < r_hi;
       c += nwarps) {
    const uint64_t r = c * 32 + lane;
    uint32_t len = 0;
    uint32_t off = 0;
    int t = 0;
    if (r >= r_lo && r < r_hi && sample_selected(rec_sample[r], rate, seed)) {
      t = lookup_table(tp.sorted_ids, tp.sorted_idx, tp.J, rec_table[r]);
      if (t < 0) {
        atomicOr(err, kErrUnknownTable);
        t = 0;
      } else {
        len = rec_len[r];
        off = uint32_t(rec_offset[r]);  // < 2^32 ids per call (checked on the host)
        if (count_records) {
          if (use_sm) {
            atomicAdd(&pres_s[t], 1u);
            atomicAdd(&acc_s[t], len);
          } else {
            atomicAdd(&present[t], 1ull);
            atomicAdd(&accesses[t], (unsigned long long)len);
          }
        }
        if (uint32_t(t) < tp.t_lo || uint32_t(t) >= tp.t_hi) len = 0;
      }
    }
    const uint32_t incl = warp_incl_scan(len);
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = incl - len;
    for (uint32_t w0 = 0; w0 < total; w0 += kWin) {
      const uint32_t w1 = min(total, w0 + uint32_t(kWin));
      // expand: record k's ids inside [w0, w1)
      __syncwarp();
      for (int k = 0; k < 32; ++k) {
        const uint32_t ek = __shfl_sync(0xffffffffu, excl, k);
        const uint32_t lk = __shfl_sync(0xffffffffu, len, k);
        const uint32_t ok = __shfl_sync(0xffffffffu, off, k);
        const int tk = __shfl_sync(0xffffffffu, t, k);
        const uint32_t s = max(ek, w0), e = min(ek + lk, w1);
        for (uint32_t q = s + lane; q < e; q += 32) {
          wtab[q - w0] = uint32_t(tk);
          wsrc[q - w0] = ok + (q - ek);
        }
      }
      __syncwarp();
      // all of the window's id loads in flight, then the counts
      constexpr int IPW = kWin / 32;
      uint32_t addr[IPW];
      bool ok[IPW];
#pragma unroll
      for (int u = 0; u < IPW; ++u) {
        const uint32_t q = w0 + lane + 32 * u;
        ok[u] = q < w1;
        addr[u] = 0;
        if (ok[u]) {
          const uint32_t tk = wtab[q - w0];
          const uint32_t idx = wsrc[q - w0];
          const uint64_t H = tp.hsize[tk];
          uint64_t row;
          if (RAW) row = fast_mod(mix64(ld_stream_u64(raw + idx)), H, tp.magic[tk]);
          else row = ld_stream_u32(ids + idx);
          if (row >= H) {
            atomicOr(err, kErrRowRange);
            ok[u] = false;
          } else {
            addr[u] = uint32_t(tp.base[tk] + row);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < IPW; ++u) {
        if (!ok[u]) continue;
        if (HOT) {
          uint32_t h = hot_hash(addr[u]);
          while (true) {
            const uint32_t kk = hkeys[h];
            if (kk == addr[u]) {
              atomicAdd(&hvals[h], 1u);
              break;
            }
            if (kk == kHotEmpty) {
              atomicAdd(&counters[addr[u]], 1u);
              break;
            }
            h = (h + 1) & (kHotSlots - 1);
          }
        } else {
          atomicAdd(&counters[addr[u]], 1u);
        }
      }
    }
  }
  if (HOT) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kHotSlots; i += blockDim.x)
      if (hvals[i]) atomicAdd(&counters[hkeys[i]], hvals[i]);
  }
  if (use_sm) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < tp.J; i += blockDim.x) {
      if (pres_s[i]) atomicAdd(&present[i], (unsigned long long)pres_s[i]);
      if (acc_s[i]) atomicAdd(&accesses[i], (unsigned long long)acc_s[i]);
    }
  }
}

// ------------------------------------------------------------------ K1, partitioned
// Large calls whose records tile the id pool contiguously (the reference
// generator's layout and every trace built by kjt_to_trace) avoid global
// atomics altogether:
//   P0  per record: info = table index (or kSkip if not selected / not in the
//       group), present/accesses counted per CTA in shared memory
//   P1  id tiles (CTA per contiguous id range): expand ids -> row address ->
//       bucket (address >> bbits); per-CTA bucket counts -> matrix[b][cta]
//   scan of the bucket-major matrix (bucket regions, per-CTA sub-regions)
//   P2  same expansion; each id's address appended to its (bucket, CTA)
//       sub-region (shared-memory cursors, only the tile's active buckets)
//   P3  CTA per (bucket, chunk): histogram of the chunk's addresses in shared
//       memory (the Zipf head contends only within one SM), flushed to the
//       global counters once
// With few buckets (<= 1024, e.g. 8 x 1e6 rows) P1 and the scan are skipped:
// P2 appends each tile's bucket runs to chunks taken from one pool
// (part_pool_kernel) and P3 reads each bucket's chunk list, so every id is
// read once.
// The expansion maps ids to records with a per-tile shared-memory window of
// record offsets (a thread per record marks the threads whose first id it
// holds, then each thread walks forward), so ids are read 8 per thread with
// vector loads.  Counts are exact integers in any order.
constexpr uint32_t kSkip = 0xFFFFFFFFu;
constexpr int kPThreads = 256;
constexpr int kPIds = 8;                         // ids per thread per tile
constexpr int kPTile = kPThreads * kPIds;        // 2048 ids
constexpr uint32_t kPMaxBuckets = 8192;  // P2: cursors + tile counts + offsets in shared memory (3 x 4 B per bucket)
constexpr int kP3Bits = 15;                      // 32768 counters per bucket (P3 shared histogram)

// P0: contiguity check + per-record info.  bad |= 1 if the records do not
// tile [0, N) in order.
__global__ void __launch_bounds__(256)
rec_info_kernel(const uint64_t* __restrict__ rec_sample, const uint32_t* __restrict__ rec_table,
                const uint64_t* __restrict__ rec_offset, const uint32_t* __restrict__ rec_len, uint64_t R,
                uint64_t N, Tables tp, double rate, uint64_t seed, bool count_records,
                uint32_t* __restrict__ roff, uint32_t* __restrict__ rinfo,
                unsigned long long* __restrict__ present, unsigned long long* __restrict__ accesses,
                unsigned* __restrict__ bad, unsigned* __restrict__ err) {
  extern __shared__ uint32_t pa[];
  const bool use_sm = count_records && tp.J <= kMaxSmemTables;
  if (use_sm)
    for (uint32_t i = threadIdx.x; i < 2 * tp.J; i += blockDim.x) pa[i] = 0;
  __syncthreads();
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < R; r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t off = rec_offset[r];
    const uint32_t len = rec_len[r];
    const uint64_t nxt = r + 1 < R ? rec_offset[r + 1] : N;
    if (off + len != nxt || (r == 0 && off != 0)) atomicOr(bad, 1u);
    roff[r] = uint32_t(off);
    uint32_t info = kSkip;
    if (sample_selected(rec_sample[r], rate, seed)) {
      const int t = lookup_table(tp.sorted_ids, tp.sorted_idx, tp.J, rec_table[r]);
      if (t < 0) {
        atomicOr(err, kErrUnknownTable);
      } else {
        if (count_records) {
          if (use_sm) {
            atomicAdd(&pa[t], 1u);
            atomicAdd(&pa[tp.J + t], len);
          } else {
            atomicAdd(&present[t], 1ull);
            atomicAdd(&accesses[t], (unsigned long long)len);
          }
        }
        if (uint32_t(t) >= tp.t_lo && uint32_t(t) < tp.t_hi && len) info = uint32_t(t);
      }
    }
    rinfo[r] = info;
  }
  if (use_sm) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < tp.J; i += blockDim.x) {
      if (pa[i]) atomicAdd(&present[i], (unsigned long long)pa[i]);
      if (pa[tp.J + i]) atomicAdd(&accesses[i], (unsigned long long)pa[tp.J + i]);
    }
  }
}

constexpr uint32_t kPSmemTables = 512;  // per-table (base, H) held in shared memory up to this J

template <int IDS>
struct alignas(16) PSmemT {
  static constexpr int kTile = kPThreads * IDS;
  static constexpr int kWin = kTile + 1;  // record window (len-1 records)
  uint32_t woff[kWin + 1];  // record offsets of the window (+ end sentinel)
  uint32_t winfo[kWin];
  uint32_t rec_of[kPThreads];   // window record holding each thread's first id
  uint32_t r0, nrec;
  uint32_t tbase[kPSmemTables];  // group-local counter base of table index t (< 2^31)
  uint32_t thash[kPSmemTables];  // its hash size
};
using PSmem = PSmemT<kPIds>;


// Loads the per-table (base, H) of the launch's tables into shared memory
// (the expansion otherwise reads both from global memory for every id).
template <class SM>
__device__ __forceinline__ void load_table_params(const Tables& tp, SM& sm) {
  if (tp.J > kPSmemTables) return;
  for (uint32_t t = threadIdx.x; t < tp.J; t += blockDim.x) {
    sm.tbase[t] = uint32_t(tp.base[t]);
    sm.thash[t] = uint32_t(tp.hsize[t]);
  }
}

// Expands tile [a, a + kPTile) of the id pool: fn(addr) for every selected id
// of an in-group table.  *rcur: first record of the tile (advanced to the
// first record of the next tile).
template <bool RAW, int IDS = kPIds, class Fn>
__device__ __forceinline__ void expand_tile(uint64_t a, uint64_t N, uint64_t R, const uint32_t* __restrict__ roff,
                                            const uint32_t* __restrict__ rinfo, const uint32_t* __restrict__ ids,
                                            const uint64_t* __restrict__ raw, const Tables& tp, PSmemT<IDS>& sm,
                                            uint32_t& rcur, unsigned* __restrict__ err, unsigned* __restrict__ bad,
                                            Fn&& fn) {
  const uint64_t tend = min(N, a + PSmemT<IDS>::kTile);
  // record window: records from rcur covering [a, tend), loaded 256 at a time
  const uint32_t r0 = rcur;
  uint32_t nwin = 0;
  while (true) {
    const uint32_t i = nwin + threadIdx.x;
    const bool in = i < uint32_t(PSmemT<IDS>::kWin) && r0 + i < R;
    uint32_t o = 0;
    if (in) {
      o = roff[r0 + i];
      sm.woff[i] = o;
      sm.winfo[i] = rinfo[r0 + i];
    }
    const uint32_t got = uint32_t(min(uint64_t(blockDim.x), min(uint64_t(PSmemT<IDS>::kWin) - nwin, R - r0 - nwin)));
    // done once a loaded record starts at or beyond the tile end
    const int covered = __syncthreads_or(in && o >= tend);
    nwin += got;
    if (covered || r0 + nwin >= R) break;
    if (nwin >= uint32_t(PSmemT<IDS>::kWin)) {  // > 2048 empty records in one tile: caller falls back
      if (threadIdx.x == 0) atomicOr(bad, 2u);
      break;
    }
  }
  // owner record of every thread's first id (thread t's ids start at a + t *
  // IDS): a thread per window record writes the slots its ids cover, and the
  // record holding id tend (the next tile's first record) names itself; the
  // last record's thread also writes the end sentinel woff[nwin]
  for (uint32_t k = threadIdx.x; k < nwin; k += blockDim.x) {
    const uint32_t lo = sm.woff[k];
    uint32_t hi;
    if (k + 1 < nwin) {
      hi = sm.woff[k + 1];
    } else {
      hi = r0 + nwin < R ? roff[r0 + nwin] : uint32_t(N);
      sm.woff[nwin] = hi;
    }
    const uint32_t s0 = lo > a ? (lo - uint32_t(a) + IDS - 1) / IDS : 0u;
    const uint32_t s1 = hi > a ? min(uint32_t(kPThreads), (min(hi, uint32_t(tend)) - uint32_t(a) + IDS - 1) / IDS) : 0u;
    for (uint32_t t = s0; t < s1; ++t) sm.rec_of[t] = k;
    if (lo <= tend && (k + 1 == nwin || hi > tend)) sm.nrec = r0 + k;
  }
  __syncthreads();
  // ids of this thread: q0 .. q0 + IDS
  const uint64_t q0 = a + uint64_t(threadIdx.x) * IDS;
  uint32_t idv[IDS];
  uint64_t rawv[RAW ? IDS : 1];
  if (q0 + IDS <= tend) {
    if (RAW) {
#pragma unroll
      for (int u = 0; u < IDS; ++u) rawv[u] = ld_stream_u64(raw + q0 + u);
    } else {
      const uint4* p = reinterpret_cast<const uint4*>(ids + q0);
#pragma unroll
      for (int v = 0; v < IDS / 4; ++v) {
        const uint4 x = __ldcs(p + v);
        idv[4 * v] = x.x;
        idv[4 * v + 1] = x.y;
        idv[4 * v + 2] = x.z;
        idv[4 * v + 3] = x.w;
      }
    }
  } else {
#pragma unroll
    for (int u = 0; u < IDS; ++u) {
      if (q0 + u < tend) {
        if (RAW) rawv[u] = raw[q0 + u];
        else idv[u] = ids[q0 + u];
      }
    }
  }
  if (q0 < tend) {
    // the current record's end, table, hash size and counter base in
    // registers, refreshed only when an id crosses into the next record
    // (one shared-memory walk step per record instead of per id)
    uint32_t k = min(sm.rec_of[threadIdx.x], nwin - 1);
    const bool smt = tp.J <= kPSmemTables;
    uint32_t rend = sm.woff[k + 1];  // woff[nwin] is the end sentinel (>= tend)
    uint32_t t = sm.winfo[k];
    uint64_t H = 0, tb = 0;
    if (t != kSkip) {
      H = smt ? sm.thash[t] : tp.hsize[t];
      tb = smt ? sm.tbase[t] : tp.base[t];
    }
#pragma unroll
    for (int u = 0; u < IDS; ++u) {
      const uint64_t q = q0 + u;
      if (q < tend) {
        if (q >= rend) {
          do {
            ++k;
            rend = k + 1 <= nwin ? sm.woff[k + 1] : uint32_t(tend);
          } while (q >= rend && k + 1 <= nwin);
          t = sm.winfo[k];
          if (t != kSkip) {
            H = smt ? sm.thash[t] : tp.hsize[t];
            tb = smt ? sm.tbase[t] : tp.base[t];
          }
        }
        if (t != kSkip) {
          const uint64_t row = RAW ? fast_mod(mix64(rawv[u]), H, tp.magic[t]) : uint64_t(idv[u]);
          if (row >= H) atomicOr(err, kErrRowRange);
          else fn(uint32_t(tb + row), u);
        }
      }
    }
  }
  // the next tile starts in the record holding id tend (named above)
  __syncthreads();
  rcur = sm.nrec;
}

// First record of id a: largest r with roff[r] <= a.
__device__ __forceinline__ uint32_t find_record(const uint32_t* __restrict__ roff, uint64_t R, uint64_t a) {
  uint64_t lo = 0, hi = R;
  while (lo + 1 < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (roff[mid] <= a) lo = mid;
    else hi = mid;
  }
  return uint32_t(lo);
}

// P1: bucket counts per CTA -> mat[b * nct + cta].
template <bool RAW>
__global__ void __launch_bounds__(kPThreads)
part_count_kernel(const uint32_t* __restrict__ roff, const uint32_t* __restrict__ rinfo, uint64_t R, uint64_t N,
                  const uint32_t* __restrict__ ids, const uint64_t* __restrict__ raw, Tables tp, uint32_t nb,
                  uint64_t ids_per_cta, uint32_t* __restrict__ mat, unsigned* __restrict__ err,
                  unsigned* __restrict__ bad) {
  __shared__ PSmem sm;
  extern __shared__ uint32_t cnt[];  // [nb]
  const uint32_t nct = gridDim.x;
  load_table_params(tp, sm);
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) cnt[i] = 0u;
  const uint64_t a0 = uint64_t(blockIdx.x) * ids_per_cta;
  const uint64_t a1 = min(N, a0 + ids_per_cta);
  if (threadIdx.x == 0 && a0 < a1) sm.nrec = find_record(roff, R, a0);
  __syncthreads();
  uint32_t rcur = sm.nrec;
  for (uint64_t a = a0; a < a1; a += kPTile)
    expand_tile<RAW>(a, a1, R, roff, rinfo, ids, raw, tp, sm, rcur, err, bad,
                     [&](uint32_t addr, int) { atomicAdd(&cnt[addr >> kP3Bits], 1u); });
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) mat[uint64_t(i) * nct + blockIdx.x] = cnt[i];
}

// P2 of the two-pass partition: each tile's addresses are counting-sorted by
// bucket in shared memory and written as contiguous per-bucket runs at the
// CTA's cursors (from the scanned P1 matrix).  Only the buckets the tile
// touches are scanned and advanced (an active list built by the first id of
// each bucket), so a tile costs O(its ids), not O(nb): with thousands of
// buckets (RM1: 6927) the per-bucket loops were the whole kernel.  Shared
// state is 8 B per bucket (cursor u32, tile count u16, active slot u16), so
// two CTAs fit per SM at 8192 buckets.
template <bool RAW>
__global__ void __launch_bounds__(kPThreads, 2)
part_scatter_kernel(const uint32_t* __restrict__ roff, const uint32_t* __restrict__ rinfo, uint64_t R, uint64_t N,
                    const uint32_t* __restrict__ ids, const uint64_t* __restrict__ raw, Tables tp, uint32_t nb,
                    uint64_t ids_per_cta, const uint32_t* __restrict__ mat, uint16_t* __restrict__ out,
                    unsigned* __restrict__ err, unsigned* __restrict__ bad) {
  __shared__ PSmem sm;
  extern __shared__ uint32_t cur[];                               // [nb] output cursors
  uint32_t* tcs = cur + nb;                                       // [nb] (tile count u16 | active slot << 16)
  __shared__ uint32_t act[kPTile];                                // active buckets; after the scan: run offsets
  __shared__ uint32_t abk[kPTile];                                // their bucket ids
  __shared__ uint32_t stage[kPTile];
  __shared__ uint32_t s_nact, s_total;
  const uint32_t nct = gridDim.x;
  load_table_params(tp, sm);
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
    cur[i] = mat[uint64_t(i) * nct + blockIdx.x];
    tcs[i] = 0;
  }
  if (threadIdx.x == 0) s_nact = 0;
  const uint64_t a0 = uint64_t(blockIdx.x) * ids_per_cta;
  const uint64_t a1 = min(N, a0 + ids_per_cta);
  if (threadIdx.x == 0 && a0 < a1) sm.nrec = find_record(roff, R, a0);
  __syncthreads();
  uint32_t rcur = sm.nrec;
  for (uint64_t a = a0; a < a1; a += kPTile) {
    uint32_t xa[kPIds], xr[kPIds];
#pragma unroll
    for (int u = 0; u < kPIds; ++u) xa[u] = kSkip;
    expand_tile<RAW>(a, a1, R, roff, rinfo, ids, raw, tp, sm, rcur, err, bad, [&](uint32_t addr, int u) {
      const uint32_t b = addr >> kP3Bits;
      const uint32_t r = atomicAdd(&tcs[b], 1u) & 0xFFFFu;
      if (r == 0) {  // first id of bucket b in this tile: list it
        const uint32_t slot = atomicAdd(&s_nact, 1u);
        abk[slot] = b;
        atomicOr(&tcs[b], slot << 16);
      }
      xa[u] = addr;
      xr[u] = r;
    });
    // expand_tile ends with a barrier: counts and the active list are complete
    const uint32_t nact = s_nact;
    const uint32_t per = (nact + blockDim.x - 1) / blockDim.x;
    uint32_t part = 0;
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t i = threadIdx.x * per + j;
      if (i < nact) part += tcs[abk[i]] & 0xFFFFu;
    }
    uint32_t tot;
    uint32_t run = block_excl_scan<uint32_t, kPThreads>(part, tot);
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t i = threadIdx.x * per + j;
      if (i < nact) {
        act[i] = run;
        run += tcs[abk[i]] & 0xFFFFu;
      }
    }
    if (threadIdx.x == 0) s_total = tot;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPIds; ++u)
      if (xa[u] != kSkip) stage[act[tcs[xa[u] >> kP3Bits] >> 16] + xr[u]] = xa[u];
    __syncthreads();
    const uint32_t total = s_total;
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
      const uint32_t x = stage[i];
      const uint32_t b = x >> kP3Bits;
      out[cur[b] + (i - act[tcs[b] >> 16])] = uint16_t(x & ((1u << kP3Bits) - 1));  // bucket-local
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nact; i += blockDim.x) {
      const uint32_t b = abk[i];
      cur[b] += tcs[b] & 0xFFFFu;
      tcs[b] = 0;
    }
    if (threadIdx.x == 0) s_nact = 0;
    // no barrier: the next tile writes only its record window before its
    // window barrier (tcs, abk and s_nact after it; nact is in registers)
  }
}

// Single-pass partition (P2 without P1): the tile's bucket runs are appended
// to per-(CTA, bucket) chunks of kPTile addresses taken from one pool with a
// global cursor, so no bucket needs its size in advance and every id is read
// once.  Every chunk except a CTA's current one per bucket ends full; those
// are closed with their fill at the end.  Chunk records (bucket, start, fill)
// go to ch_*; bchunks[b] counts bucket b's chunks.  The pool holds at most
// N + nct * nb * kPTile addresses (one partial chunk per CTA and bucket).
constexpr uint32_t kPPoolMaxBuckets = 1024;  // 6 x 4 B of shared state per bucket
constexpr uint64_t kPoolExtraBytes = uint64_t(640) << 20;  // scratch reserved for partial chunks
#ifndef RS_POOL_IDS
#define RS_POOL_IDS 16
#endif
#ifndef RS_POOL_CTAS
#define RS_POOL_CTAS 4
#endif
constexpr int kPoolIds = RS_POOL_IDS;                         // ids per thread per tile
constexpr uint32_t kPoolChunk = kPThreads * kPoolIds;         // 4096: tile = chunk
constexpr int kPoolCtasPerSm = RS_POOL_CTAS;  // 4 at 64 registers (16 B of spill) beat 3 at 80: 5.97 -> 5.81 ms
template <bool RAW>
__global__ void __launch_bounds__(kPThreads, kPoolCtasPerSm)
part_pool_kernel(const uint32_t* __restrict__ roff, const uint32_t* __restrict__ rinfo, uint64_t R, uint64_t N,
                 const uint32_t* __restrict__ ids, const uint64_t* __restrict__ raw, Tables tp, uint32_t nb,
                 uint64_t ids_per_cta, uint16_t* __restrict__ pool, unsigned* __restrict__ pool_top,
                 uint32_t* __restrict__ ch_b, uint32_t* __restrict__ ch_s, uint32_t* __restrict__ ch_n,
                 unsigned* __restrict__ n_ch, unsigned* __restrict__ bchunks, unsigned* __restrict__ err,
                 unsigned* __restrict__ bad) {
  // 4096-id tiles: half the per-tile barriers, window and scan work per id of
  // the 2048-id tiles (the pass is instruction- and barrier-bound)
  using SM = PSmemT<kPoolIds>;
  constexpr uint32_t kTile = SM::kTile;
  __shared__ SM sm;
  // per bucket: {cur: next free pool position of the current chunk, rem: free
  // entries left in it, off: the tile's run offset, nxt: the chunk this
  // tile's run overflows into} in one 16-byte word (one shared load per id)
  extern __shared__ uint4 pbs[];
  uint32_t* tcnt = reinterpret_cast<uint32_t*>(pbs + nb);  // the tile's run lengths
  uint32_t* chid = tcnt + nb;                              // current chunk record (kSkip: none)
  // (pool position, bucket-local address) of the tile's ids in bucket order:
  // aliases the record window, dead once the expansion has ended
  static_assert(sizeof(uint32_t) * (SM::kWin + 1 + SM::kWin) >= sizeof(uint2) * kTile, "stage alias");
  uint2* stage = reinterpret_cast<uint2*>(sm.woff);
  __shared__ uint32_t s_total;
  load_table_params(tp, sm);
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
    pbs[i] = make_uint4(0, 0, 0, 0);
    chid[i] = kSkip;
    tcnt[i] = 0;
  }
  const uint64_t a0 = uint64_t(blockIdx.x) * ids_per_cta;
  const uint64_t a1 = min(N, a0 + ids_per_cta);
  if (threadIdx.x == 0 && a0 < a1) sm.nrec = find_record(roff, R, a0);
  __syncthreads();
  uint32_t rcur = sm.nrec;
  const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
  for (uint64_t a = a0; a < a1; a += kTile) {
    // this thread's ids stay in registers: address and rank within its bucket's run
    uint32_t xa[kPoolIds], xr[kPoolIds];
#pragma unroll
    for (int u = 0; u < kPoolIds; ++u) xa[u] = kSkip;
    expand_tile<RAW, kPoolIds>(a, a1, R, roff, rinfo, ids, raw, tp, sm, rcur, err, bad, [&](uint32_t addr, int u) {
      xa[u] = addr;
      xr[u] = atomicAdd(&tcnt[addr >> kP3Bits], 1u);
    });
    uint32_t part = 0;
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t b = threadIdx.x * per + j;
      if (b < nb) part += tcnt[b];
    }
    uint32_t tot;
    uint32_t run = block_excl_scan<uint32_t, kPThreads>(part, tot);
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t b = threadIdx.x * per + j;
      if (b < nb) {
        const uint32_t c = tcnt[b];
        uint4 st = pbs[b];
        st.z = run;
        run += c;
        if (c > st.y) {  // the run overflows the current chunk: open the next one
          const uint32_t base = atomicAdd(pool_top, kTile);
          const uint32_t id = atomicAdd(n_ch, 1u);
          ch_b[id] = b;
          ch_s[id] = base;
          ch_n[id] = kTile;  // full unless it is still current at the end
          atomicAdd(&bchunks[b], 1u);
          st.w = base;
          chid[b] = id;  // the old chunk (if any) ends exactly full
        }
        pbs[b] = st;
      }
    }
    if (threadIdx.x == 0) s_total = tot;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPoolIds; ++u) {
      if (xa[u] != kSkip) {
        const uint4 st = pbs[xa[u] >> kP3Bits];
        const uint32_t j = xr[u];
        stage[st.z + j] = make_uint2(j < st.y ? st.x + j : st.w + (j - st.y), xa[u] & ((1u << kP3Bits) - 1));
      }
    }
    __syncthreads();
    const uint32_t total = s_total;
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
      const uint2 e = stage[i];
      pool[e.x] = uint16_t(e.y);
    }
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t b = threadIdx.x * per + j;
      if (b < nb) {
        const uint32_t c = tcnt[b];
        uint4 st = pbs[b];
        if (c > st.y) {
          st.x = st.w + (c - st.y);
          st.y = kTile - (c - st.y);
        } else {
          st.x += c;
          st.y -= c;
        }
        pbs[b] = st;
        tcnt[b] = 0;
      }
    }
    __syncthreads();  // the next tile's record window overwrites the stage
  }
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x)
    if (chid[b] != kSkip) ch_n[chid[b]] = kTile - pbs[b].y;
}

// Chunk lists per bucket: list[bstart[b] + k] = the k-th chunk of bucket b
// (any order; counts do not depend on it).  cur[] starts as bstart[].
__global__ void part_pool_list_kernel(const uint32_t* __restrict__ ch_b, const unsigned* __restrict__ n_ch,
                                      unsigned* __restrict__ cur, uint32_t* __restrict__ list) {
  const unsigned n = *n_ch;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    list[atomicAdd(&cur[ch_b[i]], 1u)] = i;
}

// Work items per bucket: ceil(chunks / per_item).
__global__ void part_pool_items_kernel(const unsigned* __restrict__ bchunks, uint32_t nb, uint32_t per_item,
                                       uint32_t* __restrict__ nitem) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) nitem[b] = (bchunks[b] + per_item - 1) / per_item;
}

// P3 over the pool: CTA per (bucket, run of per_item chunks of its list), warp
// per chunk; histogram in shared memory, flushed once.
__global__ void __launch_bounds__(1024)
part_pool_hist_kernel(const uint16_t* __restrict__ pool, const uint32_t* __restrict__ ch_s,
                      const uint32_t* __restrict__ ch_n, const uint32_t* __restrict__ list,
                      const uint32_t* __restrict__ lstart, const uint32_t* __restrict__ ibase, uint32_t nb,
                      uint32_t per_item, uint32_t* __restrict__ counters, uint64_t ncounters) {
  extern __shared__ uint32_t h[];
  constexpr uint32_t span = 1u << kP3Bits;
  const uint32_t total = ibase[nb];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
    uint32_t lo = 0, hi = nb;  // largest b with ibase[b] <= w (non-empty buckets only)
    while (lo + 1 < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (ibase[mid] <= w) lo = mid;
      else hi = mid;
    }
    while (lo + 1 < nb && ibase[lo + 1] <= w) ++lo;
    const uint32_t b = lo, c = w - ibase[lo];
    for (uint32_t i = threadIdx.x; i < span; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t k0 = lstart[b] + c * per_item, k1 = min(lstart[b + 1], k0 + per_item);
    for (uint32_t k = k0 + warp; k < k1; k += nw) {
      const uint32_t ch = list[k];
      const uint32_t s = ch_s[ch], n = ch_n[ch];  // s is a multiple of kPoolChunk: 16-byte aligned
      const uint4* p = reinterpret_cast<const uint4*>(pool + s);
      constexpr int V = 8;  // uint4 (8 addresses each) per lane in flight
#pragma unroll 1
      for (uint32_t h0 = 0; h0 < n; h0 += V * 32 * 8) {
        uint4 x[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const uint32_t e = h0 + (v * 32 + lane) * 8;
          x[v] = e < n ? __ldcs(p + (h0 >> 3) + v * 32 + lane) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const uint32_t e = h0 + (v * 32 + lane) * 8;
          const uint32_t wv[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (e + 2 * q < n) atomicAdd(&h[wv[q] & 0xFFFFu], 1u);
            if (e + 2 * q + 1 < n) atomicAdd(&h[wv[q] >> 16], 1u);
          }
        }
      }
    }
    __syncthreads();
    const uint64_t cb = uint64_t(b) << kP3Bits;
    if (ibase[b + 1] - ibase[b] == 1) {  // the bucket's only work item: plain coalesced stores
      for (uint32_t i = threadIdx.x; i < span; i += blockDim.x)
        if (cb + i < ncounters) counters[cb + i] = h[i];
    } else {
      for (uint32_t i = threadIdx.x; i < span; i += blockDim.x)
        if (h[i] && cb + i < ncounters) atomicAdd(&counters[cb + i], h[i]);
    }
    __syncthreads();
  }
}

// bstart[b] = scanned[b * nct] (first position of bucket b), bstart[nb] = total.
__global__ void part_bstart_kernel(const uint32_t* __restrict__ scanned, uint32_t nb, uint32_t nct,
                                   const uint32_t* __restrict__ total, uint32_t* __restrict__ bstart) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) bstart[b] = scanned[uint64_t(b) * nct];
  if (b == nb) bstart[nb] = *total;
}

// Chunks of each bucket for P3: nchk[b] = ceil(len_b / chunk).
__global__ void part_chunks_kernel(const uint32_t* __restrict__ bstart, uint32_t nb, uint32_t chunk,
                                   uint32_t* __restrict__ nchk) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) nchk[b] = (bstart[b + 1] - bstart[b] + chunk - 1) / chunk;
}

// P3: CTA per (bucket, chunk of the bucket's addresses); bstart[b] = first
// position of bucket b (bstart[nb] = total), cbase = exclusive scan of the
// chunk counts (cbase[nb] = total chunks).
__global__ void __launch_bounds__(1024)
part_hist_kernel(const uint16_t* __restrict__ addrs, const uint32_t* __restrict__ bstart,
                 const uint32_t* __restrict__ cbase, uint32_t nb, uint32_t chunk,
                 uint32_t* __restrict__ counters, uint64_t ncounters) {
  extern __shared__ uint32_t h[];
  constexpr uint32_t span = 1u << kP3Bits;
  const uint32_t total = cbase[nb];
  for (uint32_t w = blockIdx.x; w < total; w += gridDim.x) {
    uint32_t lo = 0, hi = nb;  // largest b with cbase[b] <= w (non-empty buckets only)
    while (lo + 1 < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (cbase[mid] <= w) lo = mid;
      else hi = mid;
    }
    while (lo + 1 < nb && cbase[lo + 1] <= w) ++lo;
    const uint32_t b = lo, c = w - cbase[lo];
    for (uint32_t i = threadIdx.x; i < span; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t p0 = bstart[b] + c * chunk;
    const uint32_t p1 = min(bstart[b + 1], p0 + chunk);
    // 8 address loads in flight per thread (two 16-bit bucket-local
    // addresses per 32-bit load), then their atomics
    constexpr int U = 8;
    const uint32_t* a32 = reinterpret_cast<const uint32_t*>(addrs);
    uint32_t q = p0;
    if ((q & 1) && q < p1) {  // odd head: one 16-bit address
      if (threadIdx.x == 0) atomicAdd(&h[addrs[q]], 1u);
      ++q;
    }
    const uint32_t w0 = q >> 1, w1 = p1 >> 1;  // whole 32-bit words [w0, w1)
    for (uint32_t pb = w0; pb < w1; pb += U * blockDim.x) {
      uint32_t x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t p = pb + u * blockDim.x + threadIdx.x;
        x[u] = p < w1 ? __ldcs(a32 + p) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pb + u * blockDim.x + threadIdx.x < w1) {
          atomicAdd(&h[x[u] & 0xFFFFu], 1u);
          atomicAdd(&h[x[u] >> 16], 1u);
        }
    }
    if ((p1 & 1) && p1 > q && threadIdx.x == 0) atomicAdd(&h[addrs[p1 - 1]], 1u);  // odd tail
    __syncthreads();
    const uint64_t cb = uint64_t(b) << kP3Bits;
    if (cbase[b + 1] - cbase[b] == 1) {  // the bucket's only work item: plain coalesced stores
      for (uint32_t i = threadIdx.x; i < span; i += blockDim.x)
        if (cb + i < ncounters) counters[cb + i] = h[i];
    } else {
      for (uint32_t i = threadIdx.x; i < span; i += blockDim.x)
        if (h[i] && cb + i < ncounters) atomicAdd(&counters[cb + i], h[i]);
    }
    __syncthreads();
  }
}

// Hot-set selection after the sample phase: rows with count >= thr (group-local
// addresses), appended up to kHotMax.
__global__ void hot_select(const uint32_t* __restrict__ counters, uint64_t n, uint32_t thr,
                          uint32_t* __restrict__ hot_list, unsigned* __restrict__ n_hot) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (counters[i] >= thr) {
      const unsigned k = atomicAdd(n_hot, 1u);
      if (k < unsigned(kHotMax)) hot_list[k] = uint32_t(i);
    }
  }
}

// K0 — batched hash_value.
__global__ void hash_ids_kernel(const uint64_t* __restrict__ raw, uint64_t n, uint64_t H,
                                uint64_t magic, uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = uint32_t(fast_mod(mix64(raw[i]), H, magic));
}

// ------------------------------------------------------------------ distinct raw ids
// GenStats.distinct_raw_ids (core/src/workload.cpp:195-223, an unordered_set
// per table) on the GPU: one open-addressing hash set of raw u64 values per
// table (capacity a power of two >= 2x the table's ids), linear probing with
// atomicCAS; successful inserts are counted.  Exact, order-independent.
constexpr uint64_t kEmpty = ~0ull;

// Per-table id totals over ALL records (the generator counts every sample).
__global__ void ids_per_table(const uint32_t* __restrict__ rec_table, const uint32_t* __restrict__ rec_len,
                              uint64_t R, const uint32_t* __restrict__ sid, const uint32_t* __restrict__ six,
                              uint32_t J, unsigned long long* __restrict__ out, unsigned* __restrict__ err) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < R;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const int t = lookup_table(sid, six, J, rec_table[r]);
    if (t < 0) atomicOr(err, kErrUnknownTable);
    else atomicAdd(&out[t], (unsigned long long)rec_len[r]);
  }
}

__global__ void __launch_bounds__(kHistThreads)
distinct_raw_kernel(const uint32_t* __restrict__ rec_table, const uint64_t* __restrict__ rec_offset,
                    const uint32_t* __restrict__ rec_len, uint64_t R, const uint64_t* __restrict__ raw,
                    const uint32_t* __restrict__ sid, const uint32_t* __restrict__ six, uint32_t J,
                    const uint64_t* __restrict__ set_base, const uint64_t* __restrict__ set_mask,
                    unsigned long long* __restrict__ slots, unsigned long long* __restrict__ count,
                    unsigned* __restrict__ has_max) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t c = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c * 32 < R; c += nwarps) {
    const uint64_t r = c * 32 + lane;
    uint32_t len = 0;
    uint64_t off = 0;
    int t = 0;
    if (r < R) {
      t = lookup_table(sid, six, J, rec_table[r]);
      if (t >= 0) {
        len = rec_len[r];
        off = rec_offset[r];
      } else {
        t = 0;
      }
    }
    const uint32_t incl = warp_incl_scan(len);
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = incl - len;
    for (uint32_t p = 0; p < total; p += 32) {
      const uint32_t q = p + lane;
      int k = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t e = __shfl_sync(0xffffffffu, excl, k + step);
        if (e <= q) k += step;
      }
      const uint64_t offk = __shfl_sync(0xffffffffu, off, k);
      const uint32_t exk = __shfl_sync(0xffffffffu, excl, k);
      const int tk = __shfl_sync(0xffffffffu, t, k);
      bool inserted = false;
      if (q < total) {
        const uint64_t v = raw[offk + (q - exk)];
        if (v == kEmpty) {
          inserted = atomicOr(&has_max[tk], 1u) == 0u;
        } else {
          const uint64_t m = set_mask[tk];
          unsigned long long* s = slots + set_base[tk];
          uint64_t h = mix64(v) & m;
          while (true) {
            const unsigned long long old = atomicCAS(&s[h], kEmpty, (unsigned long long)v);
            if (old == kEmpty) {
              inserted = true;
              break;
            }
            if (old == v) break;
            h = (h + 1) & m;
          }
        }
      }
      const unsigned act = __ballot_sync(0xffffffffu, inserted);
      if (inserted) {
        const unsigned peers = __match_any_sync(act, tk);
        if ((peers & lanemask_lt()) == 0) atomicAdd(&count[tk], (unsigned long long)__popc(peers));
      }
    }
  }
}

// ------------------------------------------------------------------ K2
// Compaction of accessed rows.  Pass 1: per-tile nonzero counts + global max.
__global__ void __launch_bounds__(kScanThreads)
nz_tile_sums(const uint32_t* __restrict__ c, size_t n, uint32_t* __restrict__ sums,
             unsigned* __restrict__ maxc) {
  const size_t base = size_t(blockIdx.x) * kScanTile + size_t(threadIdx.x) * kScanItems;
  uint32_t s = 0, m = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    size_t k = base + i;
    uint32_t v = k < n ? c[k] : 0u;
    s += v != 0;
    m = max(m, v);
  }
  uint32_t tot;
  block_excl_scan<uint32_t, kScanThreads>(s, tot);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(maxc, m);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// Pass 2: scatter (key = table << cbits | (maxc - count), value = row) in row
// order, so a stable ascending sort yields (table asc, count desc, row asc).
__global__ void __launch_bounds__(kScanThreads)
nz_scatter(const uint32_t* __restrict__ c, size_t n, const uint32_t* __restrict__ tile_pre,
           const uint64_t* __restrict__ base, uint32_t J, int cbits, uint32_t maxc,
           uint32_t* __restrict__ keys, uint32_t* __restrict__ rows) {
  const size_t k0 = size_t(blockIdx.x) * kScanTile + size_t(threadIdx.x) * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    size_t k = k0 + i;
    v[i] = k < n ? c[k] : 0u;
    s += v[i] != 0;
  }
  uint32_t tot;
  uint32_t pos = block_excl_scan<uint32_t, kScanThreads>(s, tot) + tile_pre[blockIdx.x];
  if (s == 0) return;
  // table of k0 (binary search once, then walk forward)
  uint32_t lo = 0, hi = J;
  while (lo + 1 < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (base[mid] <= k0) lo = mid;
    else hi = mid;
  }
  uint32_t t = lo;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    size_t k = k0 + i;
    if (v[i]) {
      while (t + 1 < J && base[t + 1] <= k) ++t;
      keys[pos] = (cbits >= 32 ? 0u : (uint32_t(t) << cbits)) | (maxc - v[i]);
      rows[pos] = uint32_t(k - base[t]);
      ++pos;
    }
  }
}

struct CountOfKey {
  const uint32_t* keys;
  uint32_t cmask, maxc;
  __device__ __forceinline__ uint64_t operator()(size_t i) const {
    return uint64_t(maxc - (keys[i] & cmask));
  }
};

__device__ __forceinline__ uint32_t key_table(uint32_t key, int cbits) {
  return cbits >= 32 ? 0u : key >> cbits;
}

// tstart[t] = first compacted index of table t (tstart[J] = n).
__global__ void table_starts(const uint32_t* __restrict__ keys, size_t n, int cbits, uint32_t J,
                             uint64_t* __restrict__ tstart) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i <= n;
       i += size_t(gridDim.x) * blockDim.x) {
    const int prev = i == 0 ? -1 : int(key_table(keys[i - 1], cbits));
    const int cur = i == n ? int(J) : int(key_table(keys[i], cbits));
    for (int t = prev + 1; t <= cur; ++t) tstart[t] = i;
  }
}

// access_cdf[i] = double(cum_t(i)) / double(total_t), cum inclusive within table.
__global__ void cdf_kernel(const uint32_t* __restrict__ keys, size_t n, int cbits, uint32_t maxc,
                           const uint64_t* __restrict__ cum_excl, const uint64_t* __restrict__ tstart,
                           const unsigned long long* __restrict__ totals, double* __restrict__ cdf) {
  const uint32_t cmask = cbits >= 32 ? ~0u : ((1u << cbits) - 1u);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    uint32_t key = keys[i];
    uint32_t t = key_table(key, cbits);
    uint64_t cnt = maxc - (key & cmask);
    uint64_t cum = cum_excl[i] + cnt - cum_excl[tstart[t]];
    cdf[i] = double(cum) / double(totals[t]);
  }
}

// icdf[t][p] = min k : 100 * prefix(k) >= p * total  (profiler.cpp:31-45),
// found by binary search over the inclusive prefix; icdf[t][0] = 0.
__global__ void icdf_kernel(const uint64_t* __restrict__ cum_excl, const uint64_t* __restrict__ tstart,
                            const unsigned long long* __restrict__ totals, uint32_t J,
                            uint64_t* __restrict__ icdf) {
  const uint32_t t = blockIdx.x;
  const int p = threadIdx.x;
  if (t >= J || p > 100) return;
  const uint64_t total = totals[t];
  if (p == 0 || total == 0) {
    icdf[size_t(t) * 101 + p] = 0;
    return;
  }
  const uint64_t s = tstart[t], e = tstart[t + 1], c0 = cum_excl[s];
  const uint64_t need = uint64_t(p) * total;
  // smallest k in [1, e-s] with 100 * (cum_excl[s+k] - c0) >= need
  uint64_t lo = 1, hi = e - s;
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if ((cum_excl[s + mid] - c0) * 100 >= need) hi = mid;
    else lo = mid + 1;
  }
  icdf[size_t(t) * 101 + p] = lo;
}

template <class K>
inline void set_smem_attr(K kern, size_t bytes);

// K1 partitioned (P0..P3, see part_count_kernel / part_scatter_kernel / part_pool_kernel).  Returns false (nothing counted,
// record totals already taken by P0 when count_records) when the records do
// not tile the id pool; the caller then runs the atomic kernel with
// count_records = false.
inline bool part_histogram(rs_context* ctx, Scratch& scr, bool raw, const uint64_t* d_rs, const uint32_t* d_rt,
                           const uint64_t* d_ro, const uint32_t* d_rl, uint64_t R, uint64_t N,
                           const uint32_t* d_ids, const uint64_t* d_raw, const Tables& tp, double rate, uint64_t seed,
                           bool& count_records, uint32_t nb, uint32_t* d_cnt, uint64_t ncounters,
                           unsigned long long* d_pres, unsigned long long* d_acc, unsigned* d_err) {
  cudaStream_t st = ctx->stream;
  const int sms = sm_count();
  const size_t mark = scr.used;
  uint32_t* roff = scr.take<uint32_t>(R);
  uint32_t* rinfo = scr.take<uint32_t>(R);
  unsigned* d_bad = scr.take<unsigned>(1);
  RS_CUDA(cudaMemsetAsync(d_bad, 0, 4, st));
  {
    const size_t smem = count_records && tp.J <= kMaxSmemTables ? size_t(tp.J) * 8 : 0;
    set_smem_attr(rec_info_kernel, smem);
    const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((R + 255) / 256, uint64_t(sms) * 8)));
    rec_info_kernel<<<g, 256, smem, st>>>(d_rs, d_rt, d_ro, d_rl, R, N, tp, rate, seed, count_records, roff, rinfo,
                                          d_pres, d_acc, d_bad, d_err);
    RS_COUNT(1);
  }
  count_records = false;  // taken by P0
  unsigned* hbad = ctx->pinned_buf<unsigned>(1);
  RS_CUDA(cudaMemcpyAsync(hbad, d_bad, 4, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  if (*hbad) {  // records do not tile the id pool
    scr.used = mark;
    return false;
  }
  const uint32_t nct = uint32_t(sms) * 4;
  const uint64_t ids_per_cta = ((N + nct - 1) / nct + kPTile - 1) / kPTile * kPTile;
  // single pass when the pool (N addresses + one partial chunk per CTA and
  // bucket) fits the addresses' 4 B/id of scratch plus kPoolExtraBytes
  const bool no_pool = getenv("RS_PROFILE_NO_POOL") != nullptr;  // A/B and tests of the two-pass path
  const uint32_t pct = uint32_t(sms) * kPoolCtasPerSm;
  const uint64_t pool_cap = N + uint64_t(pct) * nb * kPoolChunk;
  if (!no_pool && nb <= kPPoolMaxBuckets && pool_cap * 2 <= 4 * N + kPoolExtraBytes &&
      scr.cap - scr.used >= (pool_cap + 1) / 2 * 4 + (pool_cap / kPoolChunk + 1) * 16 + (size_t(nb) + 2) * 40 + 4096 &&
      pool_cap < (uint64_t(1) << 32)) {
    const uint64_t max_ch = pool_cap / kPoolChunk + 1;
    const uint64_t pool_ids_per_cta = ((N + pct - 1) / pct + kPoolChunk - 1) / kPoolChunk * kPoolChunk;
    uint16_t* pool = reinterpret_cast<uint16_t*>(scr.take<uint32_t>((pool_cap + 1) / 2));
    uint32_t* ch_b = scr.take<uint32_t>(max_ch);
    uint32_t* ch_s = scr.take<uint32_t>(max_ch);
    uint32_t* ch_n = scr.take<uint32_t>(max_ch);
    uint32_t* list = scr.take<uint32_t>(max_ch);
    unsigned* ctr = scr.take<unsigned>(2 + nb);  // pool_top, n_ch, bchunks[nb]
    uint32_t* lstart = scr.take<uint32_t>(nb + 1);
    unsigned* lcur = scr.take<unsigned>(nb + 1);
    uint32_t* nitem = scr.take<uint32_t>(nb + 1);
    uint32_t* ibase = scr.take<uint32_t>(nb + 1);
    RS_CUDA(cudaMemsetAsync(ctr, 0, (2 + size_t(nb)) * 4, st));
    const size_t psm = size_t(nb) * 6 * 4;  // 16 B state + run length + chunk id
    auto launch = [&](auto kern) {
      set_smem_attr(kern, psm);
      kern<<<pct, kPThreads, psm, st>>>(roff, rinfo, R, N, d_ids, d_raw, tp, nb, pool_ids_per_cta, pool, ctr, ch_b,
                                        ch_s, ch_n, ctr + 1, ctr + 2, d_err, d_bad);
    };
    if (raw) launch(part_pool_kernel<true>);
    else launch(part_pool_kernel<false>);
    RS_COUNT(1);
    hbad = ctx->pinned_buf<unsigned>(3);  // the context's one pinned buffer: {bad, pool_top, n_ch}
    unsigned* hctr = hbad + 1;
    RS_CUDA(cudaMemcpyAsync(hbad, d_bad, 4, cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaMemcpyAsync(hctr, ctr, 8, cudaMemcpyDeviceToHost, st));
    ctx->sync();
    // the bounds the pool was sized by (N + one partial chunk per CTA and bucket)
    if (uint64_t(hctr[0]) > pool_cap || uint64_t(hctr[1]) > max_ch)
      throw Error(-9, "profile: partition pool overflow (" + std::to_string(hctr[0]) + " > " +
                          std::to_string(pool_cap) + " addresses or " + std::to_string(hctr[1]) + " chunks)");
    if (*hbad) {  // a tile held more than 2048 empty records: redo with the atomic kernel
      RS_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
      scr.used = mark;
      return false;
    }
    exclusive_scan<uint32_t>(ArrayIn<uint32_t>{ctr + 2}, nb, lstart, lstart + nb, scr, st);
    RS_CUDA(cudaMemcpyAsync(lcur, lstart, (size_t(nb) + 1) * 4, cudaMemcpyDeviceToDevice, st));
    part_pool_list_kernel<<<unsigned(sms) * 4, 256, 0, st>>>(ch_b, ctr + 1, lcur, list);
    constexpr uint32_t kItemChunks = (1u << 20) / kPoolChunk;  // ~1M addresses per P3 work item
    part_pool_items_kernel<<<(nb + 255) / 256, 256, 0, st>>>(ctr + 2, nb, kItemChunks, nitem);
    exclusive_scan<uint32_t>(ArrayIn<uint32_t>{nitem}, nb, ibase, ibase + nb, scr, st);
    const size_t hsm = size_t(1) << kP3Bits << 2;
    set_smem_attr(part_pool_hist_kernel, hsm);
    part_pool_hist_kernel<<<unsigned(sms), 1024, hsm, st>>>(pool, ch_s, ch_n, list, lstart, ibase, nb, kItemChunks,
                                                             d_cnt, ncounters);
    RS_COUNT(3);
    RS_LAUNCH_CHECK();
    scr.used = mark;
    return true;
  }
  uint32_t* mat = scr.take<uint32_t>(size_t(nb) * nct);
  uint32_t* mscan = scr.take<uint32_t>(size_t(nb) * nct + 1);
  const size_t psm = size_t(nb) * 4;
  if (raw) {
    set_smem_attr(part_count_kernel<true>, psm);
    part_count_kernel<true><<<nct, kPThreads, psm, st>>>(roff, rinfo, R, N, d_ids, d_raw, tp, nb, ids_per_cta, mat,
                                                         d_err, d_bad);
  } else {
    set_smem_attr(part_count_kernel<false>, psm);
    part_count_kernel<false><<<nct, kPThreads, psm, st>>>(roff, rinfo, R, N, d_ids, d_raw, tp, nb, ids_per_cta, mat,
                                                         d_err, d_bad);
  }
  RS_COUNT(1);
  RS_CUDA(cudaMemcpyAsync(hbad, d_bad, 4, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  if (*hbad) {  // a tile held more than 2048 empty records: redo with the atomic kernel
    RS_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
    RS_CUDA(cudaMemsetAsync(d_cnt, 0, ncounters * 4, st));
    scr.used = mark;
    return false;
  }
  exclusive_scan<uint32_t>(ArrayIn<uint32_t>{mat}, size_t(nb) * nct, mscan, mscan + size_t(nb) * nct, scr, st);
  uint32_t* bstart = scr.take<uint32_t>(nb + 1);
  part_bstart_kernel<<<(nb + 256) / 256, 256, 0, st>>>(mscan, nb, nct, mscan + size_t(nb) * nct, bstart);
  uint16_t* addrs = reinterpret_cast<uint16_t*>(scr.take<uint32_t>((N + 1) / 2));
  const size_t psm2 = 2 * psm;  // cursors | tile counts + active slots
  if (raw) {
    set_smem_attr(part_scatter_kernel<true>, psm2);
    part_scatter_kernel<true><<<nct, kPThreads, psm2, st>>>(roff, rinfo, R, N, d_ids, d_raw, tp, nb, ids_per_cta,
                                                             mscan, addrs, d_err, d_bad);
  } else {
    set_smem_attr(part_scatter_kernel<false>, psm2);
    part_scatter_kernel<false><<<nct, kPThreads, psm2, st>>>(roff, rinfo, R, N, d_ids, d_raw, tp, nb, ids_per_cta,
                                                              mscan, addrs, d_err, d_bad);
  }
  constexpr uint32_t kChunkAddrs = 1u << 20;
  uint32_t* nchk = scr.take<uint32_t>(nb + 1);
  uint32_t* cbase = scr.take<uint32_t>(nb + 1);
  part_chunks_kernel<<<(nb + 255) / 256, 256, 0, st>>>(bstart, nb, kChunkAddrs, nchk);
  exclusive_scan<uint32_t>(ArrayIn<uint32_t>{nchk}, nb, cbase, cbase + nb, scr, st);
  const size_t hsm = size_t(1) << kP3Bits << 2;
  set_smem_attr(part_hist_kernel, hsm);
  part_hist_kernel<<<unsigned(sms), 1024, hsm, st>>>(addrs, bstart, cbase, nb, kChunkAddrs, d_cnt, ncounters);
  RS_COUNT(5);
  RS_LAUNCH_CHECK();
  scr.used = mark;
  return true;
}

// Allows `bytes` of dynamic shared memory on top of the kernel's static usage.
template <class K>
inline void set_smem_attr(K kern, size_t bytes) {
  // needed whenever static + dynamic shared memory passes the 48 KB default
  // (the partition kernels' static footprint alone is ~40 KB)
  cudaFuncAttributes fa{};
  RS_CUDA(cudaFuncGetAttributes(&fa, kern));
  if (fa.sharedSizeBytes + bytes > 48 * 1024)
    RS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

struct RankDevice {
  uint32_t* rows;     // n
  double* cdf;        // n
  uint64_t* icdf;     // J * 101
  uint64_t* tstart;   // J + 1
  size_t n;
  uint32_t split = 0;  // > 0: the (table, count) key does not fit 32 bits; rank
                       // at most `split` tables per call instead (nothing ranked)
};

inline int bits_for(uint64_t v) {  // bits needed to represent values 0..v
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

// K2 over one table group's u32 counters (table-major, h_base[J] offsets).
// totals: device per-table totals (the reference's st.total_accesses).
inline RankDevice rank_group(rs_context* ctx, Scratch& scr, const uint32_t* d_counters,
                             const std::vector<uint64_t>& h_base, uint32_t J,
                             const unsigned long long* d_totals) {
  cudaStream_t st = ctx->stream;
  const size_t n = h_base[J];
  const size_t tiles = (n + kScanTile - 1) / kScanTile;
  uint64_t* d_base = stage(h_base.data(), h_base.size(), false, scr, st);
  uint32_t* sums = scr.take<uint32_t>(tiles + 1);
  unsigned* d_max = scr.take<unsigned>(2);
  uint32_t* d_total = reinterpret_cast<uint32_t*>(d_max + 1);
  RS_CUDA(cudaMemsetAsync(d_max, 0, 2 * sizeof(unsigned), st));
  if (tiles) {
    nz_tile_sums<<<unsigned(tiles), kScanThreads, 0, st>>>(d_counters, n, sums, d_max);
    scan_sums_inplace<uint32_t>(sums, tiles, d_total, scr, st);
  }
  unsigned* h2 = ctx->pinned_buf<unsigned>(2);
  RS_CUDA(cudaMemcpyAsync(h2, d_max, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  ctx->sync();
  const uint32_t maxc = h2[0];
  const size_t nd = h2[1];
  const int cbits = std::max(1, bits_for(maxc));
  const int tbits = bits_for(J > 0 ? J - 1 : 0);
  RankDevice out{};
  if (cbits + tbits > 32) {
    // rows counted >= 2^(32 - tbits) times: fewer tables per key space
    out.split = cbits >= 32 ? 1u : (1u << (32 - cbits));
    return out;
  }

  out.n = nd;
  out.rows = scr.take<uint32_t>(nd + 1);
  out.cdf = scr.take<double>(nd + 1);
  out.icdf = scr.take<uint64_t>(size_t(J) * 101);
  out.tstart = scr.take<uint64_t>(J + 1);
  uint32_t* keys = scr.take<uint32_t>(nd + 1);
  if (tiles && nd)
    nz_scatter<<<unsigned(tiles), kScanThreads, 0, st>>>(d_counters, n, sums, d_base, J, cbits,
                                                         maxc, keys, out.rows);
  radix_sort_pairs(keys, out.rows, nd, cbits + tbits, scr, st);
  uint64_t* cum = scr.take<uint64_t>(nd + 1);
  exclusive_scan<uint64_t>(CountOfKey{keys, cbits >= 32 ? ~0u : ((1u << cbits) - 1u), maxc}, nd,
                           cum, cum + nd, scr, st);
  const int g = std::max(1, int(std::min<size_t>((nd + 255) / 256, size_t(sm_count()) * 8)));
  table_starts<<<g, 256, 0, st>>>(keys, nd, cbits, J, out.tstart);
  if (nd) cdf_kernel<<<g, 256, 0, st>>>(keys, nd, cbits, maxc, cum, out.tstart, d_totals, out.cdf);
  if (J) icdf_kernel<<<J, 128, 0, st>>>(cum, out.tstart, d_totals, J, out.icdf);
  RS_LAUNCH_CHECK();
  return out;
}

}  // namespace prof

// ------------------------------------------------------------------ host API
rs_profile* profile_run(rs_context* ctx, const rs_trace* tr, double rate, uint64_t seed) {
  using namespace prof;
  if (!tr) throw InvalidArgument("profile: trace is null");
  if (tr->num_samples < 1 || tr->num_tables == 0)  // profiler.cpp:62-63
    throw InvalidArgument("profile: trace is empty");
  if (!(rate > 0.0 && rate <= 1.0))  // profiler.cpp:64-65
    throw InvalidArgument("profile: sample_rate must be in (0, 1]");
  if ((tr->ids == nullptr) == (tr->raw_ids == nullptr))
    throw InvalidArgument("profile: exactly one of ids / raw_ids must be given");
  const uint32_t J = tr->num_tables;
  const bool raw = tr->raw_ids != nullptr;
  const bool on_dev = tr->location == RS_MEM_DEVICE;
  const uint64_t R = tr->num_records, N = tr->num_ids;
  if (N >= (uint64_t(1) << 32))
    throw InvalidArgument("profile: more than 2^32-1 ids per call (u32 row counters)");
  for (uint32_t j = 0; j < J; ++j) {
    if (tr->tables[j].hash_size < 1 || tr->tables[j].hash_size > 0x7FFFFFFFULL)
      throw InvalidArgument("profile: table hash_size must be in [1, 2^31-1]");
  }
  cudaStream_t st = ctx->stream;
  // RS_PROFILE_DEBUG=1: phase times on stderr (each phase synchronised)
  static const bool dbg = getenv("RS_PROFILE_DEBUG") != nullptr;
  auto t_0 = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!dbg) return;
    RS_CUDA(cudaStreamSynchronize(st));
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "profile %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t_0).count());
    t_0 = t;
  };
  phase("enter");

  // table-id lookup (sorted ids -> index), per-table hash params
  std::vector<uint32_t> order(J);
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(),
            [&](uint32_t a, uint32_t b) { return tr->tables[a].table_id < tr->tables[b].table_id; });
  std::vector<uint32_t> sids(J), sidx(J);
  std::vector<uint64_t> hs(J), mg(J);
  for (uint32_t i = 0; i < J; ++i) {
    sids[i] = tr->tables[order[i]].table_id;
    sidx[i] = order[i];
  }
  for (uint32_t j = 0; j < J; ++j) {
    hs[j] = tr->tables[j].hash_size;
    mg[j] = FastMod::make(hs[j]).m;
  }
  // table groups: sum(H) per group < 2^31 (u32 compaction positions / keys)
  // (splitting RM1's 2.3e8 rows into groups that fit the partitioned
  // histogram's buckets measured slower: 14.6 ms + a second result grow vs
  // 13.8 ms on the atomic kernel)
  const uint64_t gcap = 0x7FFFFFFFULL;
  std::vector<uint32_t> gstart{0};
  {
    uint64_t acc = 0;
    for (uint32_t j = 0; j < J; ++j) {
      if (acc + hs[j] > gcap && j > gstart.back()) {
        gstart.push_back(j);
        acc = 0;
      }
      acc += hs[j];
    }
    gstart.push_back(J);
  }
  uint64_t maxH = 0, minH = ~uint64_t(0);
  for (size_t g = 0; g + 1 < gstart.size(); ++g) {
    uint64_t s = 0;
    for (uint32_t j = gstart[g]; j < gstart[g + 1]; ++j) s += hs[j];
    maxH = std::max(maxH, s);
    minH = std::min(minH, s);
  }
  // scratch for the single-pass pool's partial chunks only when some group
  // can take that path (few buckets, a partitioned-size call): a huge table
  // set (RM3) keeps its arena as before
  const bool pool_possible = N >= (uint64_t(1) << 22) &&
                             ((minH + (uint64_t(1) << kP3Bits) - 1) >> kP3Bits) <= kPPoolMaxBuckets;

  size_t need = Scratch::bytes_for(R, 8) * 2 + Scratch::bytes_for(R, 4) * 2 +
                Scratch::bytes_for(N, raw ? 8 : 4) + Scratch::bytes_for(J, 8) * 8 +
                Scratch::bytes_for(maxH + 1, 4) * 6 + Scratch::bytes_for(maxH + 1, 8) * 3 +
                radix_sort_scratch_bytes(maxH + 1) + (size_t(J) * 101 + 4096) * 8 + (8 << 20) +
                // partitioned histogram: record info, bucket matrix, addresses
                Scratch::bytes_for(R, 4) * 2 + Scratch::bytes_for(size_t(kPMaxBuckets) * sm_count() * 4, 4) * 2 +
                Scratch::bytes_for(N, 4) + Scratch::bytes_for(kPMaxBuckets + 1, 4) * 3 +
                scan_scratch_bytes(size_t(kPMaxBuckets) * sm_count() * 4, 4) +
                // single-pass pool: chunk records and lists (the pool itself fits the addresses' N x 4 B)
                Scratch::bytes_for(N / 1024 + kPoolExtraBytes / 4096 + 2, 4) * 4 +  // chunk records (>= 2048 addresses each)
                Scratch::bytes_for(kPPoolMaxBuckets + 2, 4) * 5 + (pool_possible ? kPoolExtraBytes : 0);
  Scratch scr = ctx->scratch(need);
  phase("scratch");

  const uint64_t* d_rs = on_dev ? tr->rec_sample : stage(tr->rec_sample, R, false, scr, st);
  const uint32_t* d_rt = on_dev ? tr->rec_table : stage(tr->rec_table, R, false, scr, st);
  const uint64_t* d_ro = on_dev ? tr->rec_offset : stage(tr->rec_offset, R, false, scr, st);
  const uint32_t* d_rl = on_dev ? tr->rec_len : stage(tr->rec_len, R, false, scr, st);
  const uint32_t* d_ids = nullptr;
  const uint64_t* d_raw = nullptr;
  if (raw) d_raw = on_dev ? tr->raw_ids : stage(tr->raw_ids, N, false, scr, st);
  else d_ids = on_dev ? tr->ids : stage(tr->ids, N, false, scr, st);

  uint32_t* d_sids = stage(sids.data(), J, false, scr, st);
  uint32_t* d_sidx = stage(sidx.data(), J, false, scr, st);
  uint64_t* d_hs = stage(hs.data(), J, false, scr, st);
  uint64_t* d_mg = stage(mg.data(), J, false, scr, st);
  auto* d_pres = scr.take<unsigned long long>(J);
  auto* d_acc = scr.take<unsigned long long>(J);
  auto* d_sel = scr.take<unsigned long long>(1);
  auto* d_err = scr.take<unsigned>(1);
  RS_CUDA(cudaMemsetAsync(d_pres, 0, J * 8, st));
  RS_CUDA(cudaMemsetAsync(d_acc, 0, J * 8, st));
  RS_CUDA(cudaMemsetAsync(d_sel, 0, 8, st));
  RS_CUDA(cudaMemsetAsync(d_err, 0, 4, st));

  const int sms = sm_count();
  {
    unsigned g = unsigned(std::min<uint64_t>((tr->num_samples + 255) / 256, uint64_t(sms) * 8));
    count_selected<<<std::max(1u, g), 256, 0, st>>>(tr->num_samples, rate, seed, d_sel);
  }

  auto* res = new rs_profile;
  res->pool = ctx->host_pool;
  res->stream = st;
  res->J = J;
  res->table_ids.resize(J);
  res->coverage.resize(J);
  res->avg_pooling.resize(J);
  res->distinct.assign(J, 0);
  res->total.assign(J, 0);
  res->present.assign(J, 0);
  res->icdf.assign(size_t(J) * 101, 0);
  res->start.assign(J + 1, 0);
  try {
    std::vector<uint64_t> h_tot(J), h_pres(J);
    unsigned h_err = 0;
    unsigned long long h_sel = 0;
    for (size_t g = 0; g + 1 < gstart.size(); ++g) {
      const uint32_t t_lo = gstart[g], t_hi = gstart[g + 1], Jg = t_hi - t_lo;
      size_t mark = scr.used;
      std::vector<uint64_t> base_all(J, 0), base_g(Jg + 1, 0);
      for (uint32_t j = t_lo; j < t_hi; ++j) base_g[j - t_lo + 1] = base_g[j - t_lo] + hs[j];
      for (uint32_t j = t_lo; j < t_hi; ++j) base_all[j] = base_g[j - t_lo];
      uint64_t* d_base = stage(base_all.data(), J, false, scr, st);
      uint32_t* d_cnt = scr.take<uint32_t>(base_g[Jg] + 1);
      RS_CUDA(cudaMemsetAsync(d_cnt, 0, base_g[Jg] * 4, st));
      Tables tp{d_sids, d_sidx, d_base, d_hs, d_mg, J, t_lo, t_hi};
      const uint64_t warps = (R + 31) / 32;
      unsigned grid = unsigned(std::min<uint64_t>((warps + 7) / 8, uint64_t(sms) * 8));
      grid = std::max(1u, grid);
      const size_t rsm = (J <= kMaxSmemTables ? size_t(J) * 8 : 0) + size_t(2) * kHistWarps * kWin * 4;
      bool cr = g == 0;
      auto run = [&](auto kern, uint64_t lo, uint64_t hi, size_t smem, const uint32_t* hl, const unsigned* nh) {
        set_smem_attr(kern, smem);
        kern<<<grid, kHistThreads, smem, st>>>(d_rs, d_rt, d_ro, d_rl, lo, hi, d_ids, d_raw, tp, rate, seed, cr,
                                               hl, nh, d_cnt, d_pres, d_acc, d_err);
        RS_COUNT(1);
      };
      // large calls with contiguous records: the partitioned histogram
      bool done = false;
      const uint32_t nb = uint32_t((base_g[Jg] + (uint64_t(1) << kP3Bits) - 1) >> kP3Bits);
      const bool aligned = raw ? (reinterpret_cast<uintptr_t>(d_raw) % 8 == 0)
                               : (reinterpret_cast<uintptr_t>(d_ids) % 16 == 0);
      static const bool no_part = getenv("RS_PROFILE_NO_PARTITION") != nullptr;
      if (!no_part && N >= (uint64_t(1) << 22) && nb <= kPMaxBuckets && aligned && R < (uint64_t(1) << 32)) {
        done = part_histogram(ctx, scr, raw, d_rs, d_rt, d_ro, d_rl, R, N, d_ids, d_raw, tp, rate, seed, cr, nb,
                              d_cnt, base_g[Jg], d_pres, d_acc, d_err);
      }
      // otherwise two phases when the call is large enough for a sample to find the head
      const uint64_t Rs = N >= (uint64_t(1) << 22) && R >= 64 * 32 ? (R / 64 + 31) / 32 * 32 : R;
      if (done) {
      } else if (Rs < R) {
        uint32_t* d_hot = scr.take<uint32_t>(kHotMax);
        unsigned* d_nh = scr.take<unsigned>(1);
        RS_CUDA(cudaMemsetAsync(d_nh, 0, 4, st));
        if (raw) run(hash_hist<true, false>, 0, Rs, rsm, nullptr, nullptr);
        else run(hash_hist<false, false>, 0, Rs, rsm, nullptr, nullptr);
        // expected sample ids ~ N * Rs / R: rows at >= 1/32768 of the sample
        const uint32_t thr = uint32_t(std::max<uint64_t>(8, uint64_t(double(N) * double(Rs) / double(R) / 32768.0)));
        const unsigned gs = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((base_g[Jg] + 255) / 256, uint64_t(sms) * 8)));
        hot_select<<<gs, 256, 0, st>>>(d_cnt, base_g[Jg], thr, d_hot, d_nh);
        RS_COUNT(1);
        const size_t smem = 2 * kHotSlots * 4 + rsm;
        if (raw) run(hash_hist<true, true>, Rs, R, smem, d_hot, d_nh);
        else run(hash_hist<false, true>, Rs, R, smem, d_hot, d_nh);
      } else {
        if (raw) run(hash_hist<true, false>, 0, R, rsm, nullptr, nullptr);
        else run(hash_hist<false, false>, 0, R, rsm, nullptr, nullptr);
      }
      RS_LAUNCH_CHECK();
      phase("histogram");
      if (g == 0) {
        // errors, selection and per-table totals are known after the first group
        auto* hb = ctx->pinned_buf<uint64_t>(2 * size_t(J) + 2);
        RS_CUDA(cudaMemcpyAsync(hb, d_acc, J * 8, cudaMemcpyDeviceToHost, st));
        RS_CUDA(cudaMemcpyAsync(hb + J, d_pres, J * 8, cudaMemcpyDeviceToHost, st));
        RS_CUDA(cudaMemcpyAsync(hb + 2 * J, d_sel, 8, cudaMemcpyDeviceToHost, st));
        RS_CUDA(cudaMemcpyAsync(hb + 2 * J + 1, d_err, 4, cudaMemcpyDeviceToHost, st));
        ctx->sync();
        for (uint32_t j = 0; j < J; ++j) {
          h_tot[j] = hb[j];
          h_pres[j] = hb[J + j];
        }
        h_sel = hb[2 * J];
        h_err = uint32_t(hb[2 * J + 1]);
        if (h_sel == 0) throw InvalidArgument("profile: sample selected zero samples");
        if (h_err & kErrUnknownTable)
          throw OutOfRange("profile: record references a table id absent from trace.tables");
        if (h_err & kErrRowRange)
          throw InvalidArgument("profile: hashed id outside its table's hash_size");
      }
      // K2 over the group; a group whose hottest row needs more count bits
      // than the packed (table, count) key leaves is ranked in table ranges
      uint32_t step = Jg;
      for (uint32_t a = 0; a < Jg;) {
        const uint32_t b = std::min(Jg, a + step);
        std::vector<uint64_t> base_r(base_g.begin() + a, base_g.begin() + b + 1);
        for (auto& x : base_r) x -= base_g[a];
        const size_t mark_r = scr.used;
        RankDevice rk = rank_group(ctx, scr, d_cnt + base_g[a], base_r, b - a, d_acc + t_lo + a);
        if (rk.split) {
          scr.used = mark_r;
          step = std::min(step, rk.split);
          if (b - a <= step) throw Error(-9, "rank: table range split did not shrink the key");
          continue;
        }
        phase("rank-kernels");
        const uint32_t r_lo = t_lo + a, Jr = b - a;
        std::vector<uint64_t> tstart(Jr + 1);
        const size_t at = res->nd;
        res->grow(rk.n, st);
        phase("grow");
        RS_CUDA(cudaMemcpyAsync(tstart.data(), rk.tstart, (Jr + 1) * 8, cudaMemcpyDeviceToHost, st));
        RS_CUDA(cudaMemcpyAsync(res->icdf.data() + size_t(r_lo) * 101, rk.icdf,
                                size_t(Jr) * 101 * 8, cudaMemcpyDeviceToHost, st));
        if (rk.n) {
          RS_CUDA(cudaMemcpyAsync(res->rows + at, rk.rows, rk.n * 4, cudaMemcpyDeviceToHost, st));
          RS_CUDA(cudaMemcpyAsync(res->cdf + at, rk.cdf, rk.n * 8, cudaMemcpyDeviceToHost, st));
          RS_CUDA(cudaMemcpyAsync(res->d_rows + at, rk.rows, rk.n * 4, cudaMemcpyDeviceToDevice, st));
        }
        phase("rank");
        res->nd = at + rk.n;
        ctx->sync();
        phase("d2h");
        for (uint32_t j = r_lo; j < r_lo + Jr; ++j) res->distinct[j] = tstart[j - r_lo + 1] - tstart[j - r_lo];
        scr.used = mark_r;
        a = b;
      }
      if (g > 0) {
        // later groups (sum of hash sizes >= 2^31) can find out-of-range rows too
        auto* hb = ctx->pinned_buf<unsigned>(1);
        RS_CUDA(cudaMemcpyAsync(hb, d_err, 4, cudaMemcpyDeviceToHost, st));
        ctx->sync();
        if (hb[0] & kErrRowRange)
          throw InvalidArgument("profile: hashed id outside its table's hash_size");
      }
      scr.used = mark;
    }
    // assemble (tables are group-contiguous, so concatenation keeps order)
    for (uint32_t j = 0; j < J; ++j) res->start[j + 1] = res->start[j] + res->distinct[j];
    res->selected = h_sel;
    for (uint32_t j = 0; j < J; ++j) {  // profiler.cpp:114-121
      res->table_ids[j] = tr->tables[j].table_id;
      res->total[j] = h_tot[j];
      res->present[j] = h_pres[j];
      res->coverage[j] = double(h_pres[j]) / double(h_sel);
      res->avg_pooling[j] = h_pres[j] ? double(h_tot[j]) / double(h_pres[j]) : 0.0;
    }
    if (!res->d_rows) res->grow(0, st);
    ctx->sync();
    phase("assemble");
  } catch (...) {
    delete res;
    throw;
  }
  return res;
}

void hash_ids(rs_context* ctx, const uint64_t* raw, uint64_t n, uint64_t H, uint32_t* out,
              int location) {
  if (H == 0) throw InvalidArgument("hash_value: hash_size must be >= 1");
  if (H > 0xFFFFFFFFULL)
    throw InvalidArgument("hash_ids: hash_size must be < 2^32 (u32 rows)");
  if (n == 0) return;
  cudaStream_t st = ctx->stream;
  Scratch scr = ctx->scratch(location == RS_MEM_DEVICE ? 4096 : n * 12 + 4096);
  const uint64_t* d_raw = location == RS_MEM_DEVICE ? raw : stage(raw, n, false, scr, st);
  uint32_t* d_out = location == RS_MEM_DEVICE ? out : scr.take<uint32_t>(n);
  unsigned g = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(sm_count()) * 16));
  prof::hash_ids_kernel<<<g, 256, 0, st>>>(d_raw, n, H, FastMod::make(H).m, d_out);
  RS_LAUNCH_CHECK();
  if (location != RS_MEM_DEVICE) {
    RS_CUDA(cudaMemcpyAsync(out, d_out, n * 4, cudaMemcpyDeviceToHost, st));
    ctx->sync();
  }
}

// GenStats.distinct_raw_ids for a raw trace (core/src/workload.cpp:195-223):
// distinct raw values per table over every record.
void count_distinct_raw(rs_context* ctx, const rs_trace* tr, uint64_t* out) {
  using namespace prof;
  if (!tr || !tr->raw_ids) throw InvalidArgument("count_distinct_raw: trace must carry raw_ids");
  const uint32_t J = tr->num_tables;
  const bool on_dev = tr->location == RS_MEM_DEVICE;
  const uint64_t R = tr->num_records, N = tr->num_ids;
  cudaStream_t st = ctx->stream;
  std::vector<uint32_t> order(J), sids(J), sidx(J);
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(),
            [&](uint32_t a, uint32_t b) { return tr->tables[a].table_id < tr->tables[b].table_id; });
  for (uint32_t i = 0; i < J; ++i) {
    sids[i] = tr->tables[order[i]].table_id;
    sidx[i] = order[i];
  }
  Scratch s0 = ctx->scratch(Scratch::bytes_for(R, 8) + Scratch::bytes_for(R, 4) * 2 +
                            Scratch::bytes_for(N, 8) + Scratch::bytes_for(J + 1, 8) * 6 + (4 << 20));
  const uint32_t* d_rt = on_dev ? tr->rec_table : stage(tr->rec_table, R, false, s0, st);
  const uint64_t* d_ro = on_dev ? tr->rec_offset : stage(tr->rec_offset, R, false, s0, st);
  const uint32_t* d_rl = on_dev ? tr->rec_len : stage(tr->rec_len, R, false, s0, st);
  const uint64_t* d_raw = on_dev ? tr->raw_ids : stage(tr->raw_ids, N, false, s0, st);
  uint32_t* d_sid = stage(sids.data(), J, false, s0, st);
  uint32_t* d_six = stage(sidx.data(), J, false, s0, st);
  auto* d_n = s0.take<unsigned long long>(J);
  auto* d_err = s0.take<unsigned>(1);
  RS_CUDA(cudaMemsetAsync(d_n, 0, J * 8, st));
  RS_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
  const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((R + 255) / 256, uint64_t(sm_count()) * 8)));
  ids_per_table<<<g, 256, 0, st>>>(d_rt, d_rl, R, d_sid, d_six, J, d_n, d_err);
  std::vector<uint64_t> n(J + 1);
  RS_CUDA(cudaMemcpyAsync(n.data(), d_n, J * 8, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaMemcpyAsync(&n[J], d_err, 4, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  if (uint32_t(n[J])) throw OutOfRange("count_distinct_raw: record of a table absent from trace.tables");
  std::vector<uint64_t> base(J), mask(J);
  uint64_t total = 0;
  for (uint32_t j = 0; j < J; ++j) {
    uint64_t cap = 16;
    while (cap < 2 * n[j]) cap <<= 1;
    base[j] = total;
    mask[j] = cap - 1;
    total += cap;
  }
  const size_t used = s0.used;
  Scratch scr = ctx->scratch(used + Scratch::bytes_for(total, 8) + Scratch::bytes_for(J, 8) * 4 + (4 << 20));
  scr.used = used;  // the arena did not move unless it had to grow
  if (scr.base != s0.base) {
    // arena reallocated: restage everything
    scr.used = 0;
    d_rt = on_dev ? tr->rec_table : stage(tr->rec_table, R, false, scr, st);
    d_ro = on_dev ? tr->rec_offset : stage(tr->rec_offset, R, false, scr, st);
    d_rl = on_dev ? tr->rec_len : stage(tr->rec_len, R, false, scr, st);
    d_raw = on_dev ? tr->raw_ids : stage(tr->raw_ids, N, false, scr, st);
    d_sid = stage(sids.data(), J, false, scr, st);
    d_six = stage(sidx.data(), J, false, scr, st);
  }
  uint64_t* d_base = stage(base.data(), J, false, scr, st);
  uint64_t* d_mask = stage(mask.data(), J, false, scr, st);
  auto* slots = scr.take<unsigned long long>(total);
  auto* d_cnt = scr.take<unsigned long long>(J);
  auto* d_hm = scr.take<unsigned>(J);
  RS_CUDA(cudaMemsetAsync(slots, 0xFF, total * 8, st));
  RS_CUDA(cudaMemsetAsync(d_cnt, 0, J * 8, st));
  RS_CUDA(cudaMemsetAsync(d_hm, 0, J * 4, st));
  const uint64_t warps = (R + 31) / 32;
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, uint64_t(sm_count()) * 8)));
  distinct_raw_kernel<<<grid, kHistThreads, 0, st>>>(d_rt, d_ro, d_rl, R, d_raw, d_sid, d_six, J, d_base,
                                                     d_mask, slots, d_cnt, d_hm);
  RS_LAUNCH_CHECK();
  RS_CUDA(cudaMemcpyAsync(out, d_cnt, J * 8, cudaMemcpyDeviceToHost, st));
  ctx->sync();
}

uint32_t profile_tables(const rs_profile* p) { return p->J; }
uint64_t profile_selected(const rs_profile* p) { return p->selected; }
void profile_free(rs_profile* p) { delete p; }

void profile_view(const rs_profile* p, uint32_t j, rs_feature_stats* o) {
  if (j >= p->J) throw InvalidArgument("profile: table index out of range");
  o->table_id = p->table_ids[j];
  o->coverage = p->coverage[j];
  o->avg_pooling = p->avg_pooling[j];
  o->distinct_rows_accessed = p->distinct[j];
  o->total_accesses = p->total[j];
  o->icdf_steps = p->icdf.data() + size_t(j) * 101;
  o->access_cdf = p->cdf + p->start[j];
  o->rows_by_rank = p->rows + p->start[j];
  o->d_rows_by_rank = p->d_rows + p->start[j];
}

__global__ void narrow_counts(const uint64_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ out,
                              unsigned long long* __restrict__ total, unsigned* __restrict__ err) {
  uint64_t s = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t v = in[i];
    if (v > 0xFFFFFFFFULL) atomicOr(err, 1u);
    out[i] = uint32_t(v);
    s += v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(total, (unsigned long long)s);
}

void build_icdf(rs_context* ctx, const uint64_t* counts, uint64_t n, int location, uint64_t* out101) {
  cudaStream_t st = ctx->stream;
  Scratch scr = ctx->scratch(n * 40 + radix_sort_scratch_bytes(n + 1) + (8 << 20));
  const uint64_t* d_in = location == RS_MEM_DEVICE ? counts : stage(counts, n, false, scr, st);
  uint32_t* d_c = scr.take<uint32_t>(n + 1);
  auto* d_tot = scr.take<unsigned long long>(1);
  auto* d_err = scr.take<unsigned>(1);
  RS_CUDA(cudaMemsetAsync(d_tot, 0, 8, st));
  RS_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
  if (n) {
    unsigned g = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(sm_count()) * 8));
    narrow_counts<<<g, 256, 0, st>>>(d_in, n, d_c, d_tot, d_err);
    RS_LAUNCH_CHECK();
  }
  auto* hb = ctx->pinned_buf<uint64_t>(2);
  RS_CUDA(cudaMemcpyAsync(hb, d_tot, 8, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaMemcpyAsync(hb + 1, d_err, 4, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  if (hb[0] == 0) throw InvalidArgument("build_icdf: all access counts are zero");  // :52-53
  if (uint32_t(hb[1])) throw InvalidArgument("build_icdf: per-row counts must be < 2^32");
  std::vector<uint64_t> base{0, n};
  prof::RankDevice rk = prof::rank_group(ctx, scr, d_c, base, 1, d_tot);
  RS_CUDA(cudaMemcpyAsync(out101, rk.icdf, 101 * 8, cudaMemcpyDeviceToHost, st));
  ctx->sync();
}

}  // namespace rs
