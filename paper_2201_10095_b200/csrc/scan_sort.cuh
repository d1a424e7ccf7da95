// Device-wide scan and stable LSD radix sort (hand-written, sm_100a).
//
// Used by the profiler's rank stage (K2: stable sort by descending count over
// row-ascending input gives the reference's (count desc, row asc) order,
// core/src/profiler.cpp:136-139) and by the EmbeddingBag backward (K5: stable
// sort of lookups by row so each row's gradient is reduced in a fixed order).
//
// Scan: reduce-then-scan in three launches (tile sums -> single-CTA scan of
// tile sums -> tile scan + carry-in).  Radix sort: 8-bit digits, per pass
// upsweep (per-tile digit counts) -> scan of the digit-major count matrix ->
// downsweep (stable in-tile ranking with warp ballots, scatter).  No atomics
// and no inter-CTA spinning, so there is no forward-progress hazard.  The
// backward's segmented sort runs the onesweep variant at the end of the file
// (one kernel per pass, decoupled look-back over tiles claimed in order).
#pragma once

#include "common.cuh"

namespace rs {

// ----------------------------------------------------------------- scratch
// Minimal bump allocator over a caller-owned device arena.
struct Scratch {
  char* base = nullptr;
  size_t cap = 0;
  size_t used = 0;
  template <class T>
  T* take(size_t n) {
    size_t off = (used + 255) & ~size_t(255);
    size_t bytes = n * sizeof(T);
    if (off + bytes > cap)
      throw Error(-9, "scratch arena exhausted (" + std::to_string(off + bytes) +
                          " > " + std::to_string(cap) + " bytes)");
    used = off + bytes;
    return reinterpret_cast<T*>(base + off);
  }
  static size_t bytes_for(size_t n, size_t elem) { return ((n * elem + 255) & ~size_t(255)); }
};

// ----------------------------------------------------------------- scan
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total
// in `total`.  Safe to call repeatedly (trailing barrier guards the smem).
template <class T, int NT>
__device__ __forceinline__ T block_excl_scan(T v, T& total) {
  __shared__ T warp_tot[NT / 32];
  __shared__ T tot_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = lane < NT / 32 ? warp_tot[lane] : T(0);
    T xi = warp_incl_scan(x);
    if (lane < NT / 32) warp_tot[lane] = xi - x;
    if (lane == 31) tot_s = xi;
  }
  __syncthreads();
  T res = inc - v + warp_tot[w];
  total = tot_s;
  __syncthreads();
  return res;
}

// in[i] may be read through a transform (e.g. "count != 0" flags).
template <class T, class In>
__global__ void __launch_bounds__(kScanThreads) scan_tile_sums(In in, size_t n, T* tile_sums) {
  const size_t base = size_t(blockIdx.x) * kScanTile;
  T s = 0;
#pragma unroll 4
  for (int i = 0; i < kScanItems; ++i) {
    size_t k = base + size_t(i) * kScanThreads + threadIdx.x;
    if (k < n) s += T(in(k));
  }
  T tot;
  block_excl_scan<T, kScanThreads>(s, tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// Single CTA exclusive scan of tile sums (n <= 1024 * 64).
template <class T>
__global__ void __launch_bounds__(1024) scan_tile_sums_excl(T* sums, size_t n, T* grand_total) {
  const int per = int((n + 1023) / 1024);
  T loc[64];
  T s = 0;
  for (int i = 0; i < per; ++i) {
    size_t k = size_t(threadIdx.x) * per + i;
    loc[i] = k < n ? sums[k] : T(0);
    s += loc[i];
  }
  T tot;
  T pre = block_excl_scan<T, 1024>(s, tot);
  for (int i = 0; i < per; ++i) {
    size_t k = size_t(threadIdx.x) * per + i;
    if (k < n) sums[k] = pre;
    pre += loc[i];
  }
  if (threadIdx.x == 0 && grand_total) *grand_total = tot;
}

// Exclusive scan of a tile with carry-in; elements are processed in
// blocked-per-thread order so each thread owns kScanItems consecutive items.
template <class T, class In>
__global__ void __launch_bounds__(kScanThreads) scan_tiles(In in, size_t n, const T* tile_pre, T* out) {
  const size_t base = size_t(blockIdx.x) * kScanTile + size_t(threadIdx.x) * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    size_t k = base + i;
    v[i] = k < n ? T(in(k)) : T(0);
    s += v[i];
  }
  T tot;
  T pre = block_excl_scan<T, kScanThreads>(s, tot) + tile_pre[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    size_t k = base + i;
    if (k < n) out[k] = pre;
    pre += v[i];
  }
}

template <class T>
struct ArrayIn {
  const T* p;
  __device__ __forceinline__ T operator()(size_t k) const { return p[k]; }
};

inline size_t scan_scratch_bytes(size_t n, size_t elem) {
  size_t tiles = (n + kScanTile - 1) / kScanTile;
  return Scratch::bytes_for(tiles + 1, elem) * 3 + 4096;
}

template <class T, class In>
void exclusive_scan(In in, size_t n, T* out, T* total, Scratch& scr, cudaStream_t st);

// In-place exclusive scan of per-tile sums (single CTA when it fits, else
// recursively through exclusive_scan).
template <class T>
void scan_sums_inplace(T* sums, size_t tiles, T* total, Scratch& scr, cudaStream_t st) {
  if (tiles <= size_t(1024) * 64) {
    scan_tile_sums_excl<T><<<1, 1024, 0, st>>>(sums, tiles, total);
    RS_COUNT(1);
    RS_LAUNCH_CHECK();
    return;
  }
  size_t mark = scr.used;
  T* tmp = scr.take<T>(tiles);
  exclusive_scan<T>(ArrayIn<T>{sums}, tiles, tmp, total, scr, st);
  RS_CUDA(cudaMemcpyAsync(sums, tmp, tiles * sizeof(T), cudaMemcpyDeviceToDevice, st));
  scr.used = mark;
}

// out[k] = sum_{i<k} in(i); optionally *total (device) = sum of all.
template <class T, class In>
void exclusive_scan(In in, size_t n, T* out, T* total, Scratch& scr, cudaStream_t st) {
  size_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 0) {
    if (total) RS_CUDA(cudaMemsetAsync(total, 0, sizeof(T), st));
    return;
  }
  size_t mark = scr.used;
  T* sums = scr.take<T>(tiles);
  scan_tile_sums<T, In><<<unsigned(tiles), kScanThreads, 0, st>>>(in, n, sums);
  scan_sums_inplace<T>(sums, tiles, total, scr, st);
  scan_tiles<T, In><<<unsigned(tiles), kScanThreads, 0, st>>>(in, n, sums, out);
  RS_COUNT(2);
  RS_LAUNCH_CHECK();
  scr.used = mark;
}

// ----------------------------------------------------------------- radix sort
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 8;                       // rounds per warp
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048 keys per CTA
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

// Peers of this lane with the same digit (one MATCH.ANY; measured faster than
// BITS bit-split ballots on B200).
template <int BITS>
__device__ __forceinline__ unsigned digit_peers(unsigned d, bool valid) {
  const unsigned pm = __match_any_sync(0xffffffffu, valid ? d : 0xFFFFFFFFu);
  return valid ? pm : 0u;
}

// Tiles of the sort.  Default (pos == nullptr): tile b = [b*kSortTile, ..),
// counts digit-major (counts[d * ntiles + b]).  Segmented: tile b =
// [pos[b], pos[b+1]) never crosses a segment, counts laid out
// [segment][digit][tile in segment] (index cidx[b] + d * cstride[b]), so one
// global exclusive scan yields each segment's offsets and every segment is
// sorted in place.
struct TileMap {
  const uint32_t* pos = nullptr;
  const uint32_t* cidx = nullptr;
  const uint32_t* cstride = nullptr;
  const uint32_t* ntd = nullptr;  // device tile count (the grid is a capacity)
  __device__ __forceinline__ bool idle(unsigned b) const { return ntd && b >= *ntd; }
  __device__ __forceinline__ size_t begin(unsigned b) const { return pos ? pos[b] : size_t(b) * kSortTile; }
  __device__ __forceinline__ size_t end(unsigned b, size_t n) const {
    return pos ? pos[b + 1] : min(n, size_t(b + 1) * kSortTile);
  }
  __device__ __forceinline__ size_t cnt(unsigned b, unsigned d, unsigned ntiles) const {
    return pos ? size_t(cidx[b]) + size_t(d) * cstride[b] : size_t(d) * ntiles + b;
  }
};

// Per-tile digit counts (TileMap layout).
static __global__ void __launch_bounds__(kSortThreads)
radix_upsweep(const uint32_t* __restrict__ keys, size_t n, int shift, int nbits,
              uint32_t* __restrict__ counts, unsigned ntiles, TileMap tm) {
  __shared__ uint32_t wc[kSortWarps][kRadix];
  if (tm.idle(blockIdx.x)) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = lane; i < kRadix; i += 32) wc[w][i] = 0;
  __syncwarp();
  const unsigned mask = (1u << nbits) - 1u;
  const size_t tend = tm.end(blockIdx.x, n);
  const size_t wbase = tm.begin(blockIdx.x) + size_t(w) * 32 * kSortItems;
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    size_t k = wbase + size_t(r) * 32 + lane;
    bool valid = k < tend;
    unsigned d = valid ? (keys[k] >> shift) & mask : 0u;
    unsigned peers = digit_peers<kRadixBits>(d, valid);
    if (valid && (peers & lanemask_lt()) == 0) wc[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) s += wc[ww][d];
    counts[tm.cnt(blockIdx.x, d, ntiles)] = s;
  }
}

// Stable scatter: offsets[d * ntiles + tile] holds the global start of digit d
// for this tile (exclusive scan of the digit-major count matrix).
#ifndef RS_SORT_MINB
#define RS_SORT_MINB 5
#endif
template <bool HAS_VALUES>
static __global__ void __launch_bounds__(kSortThreads, RS_SORT_MINB)
radix_downsweep(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                size_t n, int shift, int nbits, const uint32_t* __restrict__ offsets,
                unsigned ntiles, uint32_t* __restrict__ keys_out,
                uint32_t* __restrict__ vals_out, TileMap tm) {
  __shared__ uint32_t wc[kSortWarps][kRadix];
  if (tm.idle(blockIdx.x)) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = lane; i < kRadix; i += 32) wc[w][i] = 0;
  __syncwarp();
  const unsigned mask = (1u << nbits) - 1u;
  const size_t tile0 = tm.begin(blockIdx.x), tend = tm.end(blockIdx.x, n);
  const size_t wbase = tile0 + size_t(w) * 32 * kSortItems;
  uint32_t kk[kSortItems], vv[kSortItems], rank[kSortItems];
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    size_t k = wbase + size_t(r) * 32 + lane;
    bool valid = k < tend;
    kk[r] = valid ? keys_in[k] : 0u;
    if (HAS_VALUES) vv[r] = valid ? vals_in[k] : 0u;
    unsigned d = (kk[r] >> shift) & mask;
    unsigned peers = digit_peers<kRadixBits>(d, valid);
    unsigned leader = peers ? __ffs(peers) - 1 : 0;
    uint32_t base = 0;
    if (valid && lane == int(leader)) base = wc[w][d];
    // every lane fetches the base from its own leader
    uint32_t b2 = __shfl_sync(0xffffffffu, base, leader);
    rank[r] = b2 + __popc(peers & lanemask_lt());
    if (valid && lane == int(leader)) wc[w][d] = base + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // Per digit: offsets of each warp inside the digit, the digit's start inside
  // the tile, and its global start.  The tile is then re-laid out in shared
  // memory in (digit, rank) order and written as contiguous per-digit runs, so
  // the global stores coalesce instead of scattering 4-byte writes.
  __shared__ uint32_t dstart[kRadix], gbase[kRadix];
  __shared__ uint32_t sk[kSortTile], sv[HAS_VALUES ? kSortTile : 1];
  static_assert(kRadix == kSortThreads, "one digit per thread");
  const int d0 = threadIdx.x;
  uint32_t cnt = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) {
    const uint32_t c = wc[ww][d0];
    wc[ww][d0] = cnt;
    cnt += c;
  }
  uint32_t tot_unused;
  const uint32_t ds = block_excl_scan<uint32_t, kSortThreads>(cnt, tot_unused);
  dstart[d0] = ds;
  gbase[d0] = offsets[tm.cnt(blockIdx.x, d0, ntiles)];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    size_t k = wbase + size_t(r) * 32 + lane;
    if (k < tend) {
      const unsigned d = (kk[r] >> shift) & mask;
      const uint32_t tp = dstart[d] + wc[w][d] + rank[r];
      sk[tp] = kk[r];
      if (HAS_VALUES) sv[tp] = vv[r];
    }
  }
  __syncthreads();
  const uint32_t tn = uint32_t(tend - tile0);
  for (uint32_t i = threadIdx.x; i < tn; i += kSortThreads) {
    const uint32_t key = sk[i];
    const unsigned d = (key >> shift) & mask;
    const uint32_t pos = gbase[d] + (i - dstart[d]);
    keys_out[pos] = key;
    if (HAS_VALUES) vals_out[pos] = sv[i];
  }
}

// extra_tiles: segmented sorts round every segment up to whole tiles
inline size_t radix_sort_scratch_bytes(size_t n, size_t extra_tiles = 0) {
  size_t tiles = (n + kSortTile - 1) / kSortTile + extra_tiles;
  size_t cnt = tiles * kRadix;
  return Scratch::bytes_for(cnt, 4) * 2 + scan_scratch_bytes(cnt, 4) +
         Scratch::bytes_for(n, 4) * 2 + 4096;
}

// Stable ascending sort of (keys, vals) on bits [0, end_bit).  Sorted data
// ends in (keys, vals) — ping-pong buffers come from scratch.  n < 2^32.
// (A one-kernel-per-pass decoupled look-back variant measured slower on B200
// RM1: 3.00 vs 2.93 ms backward.)
// With tm.ntd the tile count lives on the device (seg_tiles is the grid
// capacity, n an upper bound).  With keys_res/vals_res the result stays where
// the last pass wrote it (no copy back; it may be in scr) and they receive it.
inline void radix_sort_pairs(uint32_t* keys, uint32_t* vals, size_t n, int end_bit,
                             Scratch& scr, cudaStream_t st, TileMap tm = TileMap{}, unsigned seg_tiles = 0,
                             uint32_t** keys_res = nullptr, uint32_t** vals_res = nullptr) {
  if (keys_res) *keys_res = keys;
  if (vals_res) *vals_res = vals;
  if (n <= 1 || end_bit <= 0) return;
  if (n >= (size_t(1) << 32)) throw Error(-1, "radix_sort_pairs: n >= 2^32");
  const unsigned ntiles = tm.pos ? seg_tiles : unsigned((n + kSortTile - 1) / kSortTile);
  size_t mark = scr.used;
  uint32_t* counts = scr.take<uint32_t>(size_t(ntiles) * kRadix);
  uint32_t* offs = scr.take<uint32_t>(size_t(ntiles) * kRadix);
  uint32_t* k2 = scr.take<uint32_t>(n);
  uint32_t* v2 = vals ? scr.take<uint32_t>(n) : nullptr;
  uint32_t *ki = keys, *vi = vals, *ko = k2, *vo = v2;
  for (int shift = 0; shift < end_bit; shift += kRadixBits) {
    int nb = end_bit - shift < kRadixBits ? end_bit - shift : kRadixBits;
    radix_upsweep<<<ntiles, kSortThreads, 0, st>>>(ki, n, shift, nb, counts, ntiles, tm);
    size_t m2 = scr.used;
    exclusive_scan<uint32_t>(ArrayIn<uint32_t>{counts}, size_t(ntiles) * kRadix, offs,
                             (uint32_t*)nullptr, scr, st);
    scr.used = m2;
    if (vals)
      radix_downsweep<true><<<ntiles, kSortThreads, 0, st>>>(ki, vi, n, shift, nb, offs,
                                                             ntiles, ko, vo, tm);
    else
      radix_downsweep<false><<<ntiles, kSortThreads, 0, st>>>(ki, nullptr, n, shift, nb,
                                                              offs, ntiles, ko, nullptr, tm);
    RS_COUNT(2);
    RS_LAUNCH_CHECK();
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  if (keys_res) {
    *keys_res = ki;
    if (vals_res) *vals_res = vi;
    return;  // the result may live in scr: keep it reserved
  }
  if (ki != keys) {
    RS_CUDA(cudaMemcpyAsync(keys, ki, n * 4, cudaMemcpyDeviceToDevice, st));
    if (vals) RS_CUDA(cudaMemcpyAsync(vals, vi, n * 4, cudaMemcpyDeviceToDevice, st));
  }
  scr.used = mark;
}

// ----------------------------------------------------------------- onesweep
// Segmented LSD radix sort with one kernel per pass (decoupled look-back):
// one histogram kernel counts every pass's digits per segment (table) up
// front, a small kernel turns them into each (segment, pass, digit) start, and
// each pass kernel ranks its tile, publishes its digit counts, looks back over
// the earlier tiles OF ITS SEGMENT for their running totals, and scatters —
// instead of per pass an upsweep (a second read of the keys), a scan of the
// [segment][digit][tile] count matrix and a downsweep.  Tiles are claimed in
// order through an atomic counter, so a tile only ever waits for tiles that
// were already running (forward progress).  Same stable order as the
// upsweep/downsweep sort: results are identical.
constexpr uint32_t kOsAgg = 1u << 30, kOsInc = 2u << 30, kOsCount = (1u << 30) - 1;
constexpr int kOsMaxPasses = 4;

// First tile of tile b's segment: cidx[b] = kRadix * first + (b - first).
__device__ __forceinline__ unsigned os_first(const TileMap& tm, unsigned b) {
  return (tm.cidx[b] - b) / unsigned(kRadix - 1);
}

static __global__ void __launch_bounds__(kSortThreads)
radix_os_hist(const uint32_t* __restrict__ keys, size_t n, int end_bit, uint32_t* __restrict__ hist, TileMap tm) {
  __shared__ uint32_t h[kOsMaxPasses][kRadix];
  if (tm.idle(blockIdx.x)) return;
  const int npass = (end_bit + kRadixBits - 1) / kRadixBits;
  for (int i = threadIdx.x; i < npass * kRadix; i += blockDim.x) h[i / kRadix][i % kRadix] = 0;
  __syncthreads();
  const size_t t0 = tm.begin(blockIdx.x), t1 = tm.end(blockIdx.x, n);
  for (size_t k = t0 + threadIdx.x; k < t1; k += blockDim.x) {
    const uint32_t key = keys[k];
    for (int p = 0; p < npass; ++p) {
      const int nb = min(kRadixBits, end_bit - p * kRadixBits);
      atomicAdd(&h[p][(key >> (p * kRadixBits)) & ((1u << nb) - 1u)], 1u);
    }
  }
  __syncthreads();
  const unsigned f = os_first(tm, blockIdx.x);
  for (int i = threadIdx.x; i < npass * kRadix; i += blockDim.x) {
    const uint32_t c = h[i / kRadix][i % kRadix];
    if (c) atomicAdd(&hist[(size_t(f) * npass + i / kRadix) * kRadix + i % kRadix], c);
  }
}

// base[(first * npass + p) * 256 + d] = segment start + exclusive digit prefix.
static __global__ void __launch_bounds__(kSortThreads)
radix_os_base(const uint32_t* __restrict__ hist, int npass, uint32_t* __restrict__ base, TileMap tm) {
  if (tm.idle(blockIdx.x) || os_first(tm, blockIdx.x) != blockIdx.x) return;
  const uint32_t start = uint32_t(tm.begin(blockIdx.x));
  for (int p = 0; p < npass; ++p) {
    const size_t o = (size_t(blockIdx.x) * npass + p) * kRadix + threadIdx.x;
    uint32_t tot;
    const uint32_t x = block_excl_scan<uint32_t, kSortThreads>(hist[o], tot);
    base[o] = start + x;
  }
}

template <bool HAS_VALUES>
static __global__ void __launch_bounds__(kSortThreads, RS_SORT_MINB)
radix_os_pass(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, size_t n, int shift,
              int nbits, int pass, int npass, const uint32_t* __restrict__ base, uint32_t* __restrict__ status,
              unsigned* __restrict__ ctr, uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
              TileMap tm) {
  __shared__ uint32_t wc[kSortWarps][kRadix];
  __shared__ unsigned s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(ctr, 1u);
  __syncthreads();
  const unsigned tile = s_tile;
  if (tm.idle(tile)) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = lane; i < kRadix; i += 32) wc[w][i] = 0;
  __syncwarp();
  const unsigned mask = (1u << nbits) - 1u;
  const size_t tile0 = tm.begin(tile), tend = tm.end(tile, n);
  const size_t wbase = tile0 + size_t(w) * 32 * kSortItems;
  uint32_t kk[kSortItems], vv[kSortItems], rank[kSortItems];
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    size_t k = wbase + size_t(r) * 32 + lane;
    bool valid = k < tend;
    kk[r] = valid ? keys_in[k] : 0u;
    if (HAS_VALUES) vv[r] = valid ? vals_in[k] : 0u;
    unsigned d = (kk[r] >> shift) & mask;
    unsigned peers = digit_peers<kRadixBits>(d, valid);
    unsigned leader = peers ? __ffs(peers) - 1 : 0;
    uint32_t b0 = 0;
    if (valid && lane == int(leader)) b0 = wc[w][d];
    uint32_t b2 = __shfl_sync(0xffffffffu, b0, leader);
    rank[r] = b2 + __popc(peers & lanemask_lt());
    if (valid && lane == int(leader)) wc[w][d] = b0 + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  __shared__ uint32_t dstart[kRadix], gbase[kRadix];
  __shared__ uint32_t sk[kSortTile], sv[HAS_VALUES ? kSortTile : 1];
  const int d0 = threadIdx.x;
  uint32_t cnt = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) {
    const uint32_t c = wc[ww][d0];
    wc[ww][d0] = cnt;
    cnt += c;
  }
  // publish this tile's count of digit d0, then look back over the earlier
  // tiles of the segment for their running total
  const unsigned first = os_first(tm, tile);
  volatile uint32_t* vs = status;
  if (tile == first) {
    vs[size_t(tile) * kRadix + d0] = kOsInc | cnt;
  } else {
    vs[size_t(tile) * kRadix + d0] = kOsAgg | cnt;
  }
  uint32_t excl = 0;
  if (tile != first) {
    unsigned j = tile - 1;
    while (true) {
      const uint32_t st = vs[size_t(j) * kRadix + d0];
      if ((st & ~kOsCount) == 0) continue;  // not published yet
      excl += st & kOsCount;
      if (st & kOsInc) break;
      --j;
    }
    vs[size_t(tile) * kRadix + d0] = kOsInc | (excl + cnt);
  }
  uint32_t tot_unused;
  const uint32_t ds = block_excl_scan<uint32_t, kSortThreads>(cnt, tot_unused);
  dstart[d0] = ds;
  gbase[d0] = base[(size_t(first) * npass + pass) * kRadix + d0] + excl;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    size_t k = wbase + size_t(r) * 32 + lane;
    if (k < tend) {
      const unsigned d = (kk[r] >> shift) & mask;
      const uint32_t tp = dstart[d] + wc[w][d] + rank[r];
      sk[tp] = kk[r];
      if (HAS_VALUES) sv[tp] = vv[r];
    }
  }
  __syncthreads();
  const uint32_t tn = uint32_t(tend - tile0);
  for (uint32_t i = threadIdx.x; i < tn; i += kSortThreads) {
    const uint32_t key = sk[i];
    const unsigned d = (key >> shift) & mask;
    const uint32_t pos = gbase[d] + (i - dstart[d]);
    keys_out[pos] = key;
    if (HAS_VALUES) vals_out[pos] = sv[i];
  }
}

inline size_t radix_onesweep_scratch_bytes(size_t n, size_t seg_tiles) {
  return Scratch::bytes_for(seg_tiles * kOsMaxPasses * kRadix, 4) * 2 + Scratch::bytes_for(seg_tiles * kRadix, 4) +
         Scratch::bytes_for(n, 4) * 2 + 4096;
}

// The segmented sort (tm.pos set) through the onesweep kernels; same contract
// as radix_sort_pairs.
inline void radix_sort_pairs_onesweep(uint32_t* keys, uint32_t* vals, size_t n, int end_bit, Scratch& scr,
                                      cudaStream_t st, TileMap tm, unsigned seg_tiles, uint32_t** keys_res,
                                      uint32_t** vals_res) {
  *keys_res = keys;
  if (vals_res) *vals_res = vals;
  if (n <= 1 || end_bit <= 0) return;
  const int npass = (end_bit + kRadixBits - 1) / kRadixBits;
  if (npass > kOsMaxPasses) throw Error(-9, "radix onesweep: more than 32 key bits");
  uint32_t* hist = scr.take<uint32_t>(size_t(seg_tiles) * npass * kRadix);
  uint32_t* base = scr.take<uint32_t>(size_t(seg_tiles) * npass * kRadix);
  uint32_t* status = scr.take<uint32_t>(size_t(seg_tiles) * kRadix);
  uint32_t* ctr = scr.take<uint32_t>(kOsMaxPasses);
  uint32_t* k2 = scr.take<uint32_t>(n);
  uint32_t* v2 = vals ? scr.take<uint32_t>(n) : nullptr;
  RS_CUDA(cudaMemsetAsync(hist, 0, size_t(seg_tiles) * npass * kRadix * 4, st));
  RS_CUDA(cudaMemsetAsync(ctr, 0, kOsMaxPasses * 4, st));
  radix_os_hist<<<seg_tiles, kSortThreads, 0, st>>>(keys, n, end_bit, hist, tm);
  radix_os_base<<<seg_tiles, kSortThreads, 0, st>>>(hist, npass, base, tm);
  RS_COUNT(2);
  uint32_t *ki = keys, *vi = vals, *ko = k2, *vo = v2;
  for (int p = 0; p < npass; ++p) {
    const int shift = p * kRadixBits;
    const int nb = end_bit - shift < kRadixBits ? end_bit - shift : kRadixBits;
    RS_CUDA(cudaMemsetAsync(status, 0, size_t(seg_tiles) * kRadix * 4, st));
    if (vals)
      radix_os_pass<true><<<seg_tiles, kSortThreads, 0, st>>>(ki, vi, n, shift, nb, p, npass, base, status, ctr + p,
                                                              ko, vo, tm);
    else
      radix_os_pass<false><<<seg_tiles, kSortThreads, 0, st>>>(ki, nullptr, n, shift, nb, p, npass, base, status,
                                                               ctr + p, ko, nullptr, tm);
    RS_COUNT(1);
    RS_LAUNCH_CHECK();
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  *keys_res = ki;
  if (vals_res) *vals_res = vi;
}

}  // namespace rs
