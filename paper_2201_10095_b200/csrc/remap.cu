// K3 — remap-table construction on the GPU (core/src/remap.cpp:40-105).
//
// Row classes after scattering each ranked row's rank into `m`:
//   A  rank <  min(hbm_rows, distinct)        -> fast, offset = rank      (:67-70)
//   B  rank >= min(hbm_rows, distinct)        -> slow (accessed)
//   C  never accessed (m = 0xFFFFFFFF)        -> the first
//        extra = max(0, hbm_rows - distinct) in index order are fast,
//        offset distinct + ordinal (:71-78); the rest are slow.
// Slow offsets are ordinals in ascending row order (:97-103); with
// omit_unaccessed the B rows are numbered first, then the C rows (:85-96).
// Both ordinals come from ONE exclusive scan over packed (B << 32 | C) flags.
// Output encoding: fast v >= 0, slow -(k) - 1 (include/shardplan/remap.hpp:27-29).
#include "../../include/shardplan_gpu.h"
#include "context.cuh"

namespace rs {
namespace remap {

constexpr uint32_t kNone = 0xFFFFFFFFu;

__global__ void scatter_ranks(const uint32_t* __restrict__ rows_by_rank, uint64_t distinct,
                              uint64_t H, uint32_t* __restrict__ m, unsigned* __restrict__ err) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < distinct;
       r += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t row = rows_by_rank[r];
    if (row >= H) atomicOr(err, 1u);
    else m[row] = uint32_t(r);
  }
}

struct ClassFlags {
  const uint32_t* m;
  uint32_t ranked_fast;
  __device__ __forceinline__ uint64_t operator()(size_t i) const {
    uint32_t v = m[i];
    uint64_t b = (v != kNone && v >= ranked_fast) ? 1ull : 0ull;
    uint64_t c = v == kNone ? 1ull : 0ull;
    return (b << 32) | c;
  }
};

__global__ void finalize(const uint32_t* __restrict__ m, const uint64_t* __restrict__ ord,
                         const uint64_t* __restrict__ totals, uint64_t H, uint32_t ranked_fast,
                         uint64_t distinct, uint64_t extra, bool omit, int32_t* __restrict__ out) {
  const uint64_t nB = totals[0] >> 32;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < H;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = m[i];
    const uint64_t o = ord[i];
    const uint64_t ob = o >> 32, oc = o & 0xFFFFFFFFull;
    int32_t e;
    if (v != kNone && v < ranked_fast) {
      e = int32_t(v);
    } else if (v != kNone) {  // B: accessed, slow
      // default order interleaves B and C by row index
      uint64_t k = omit ? ob : (ob + oc - (oc < extra ? oc : extra));
      e = int32_t(-int64_t(k) - 1);
    } else if (oc < extra) {  // C promoted to the fast tier
      e = int32_t(distinct + oc);
    } else {
      uint64_t k = omit ? nB + (oc - extra) : (ob + oc - extra);
      e = int32_t(-int64_t(k) - 1);
    }
    out[i] = e;
  }
}

}  // namespace remap

void build_remap(rs_context* ctx, uint32_t table_id, uint64_t H, uint64_t hbm_rows,
                 const uint32_t* rows_by_rank, uint64_t distinct, int rows_location, int omit,
                 int32_t* entries, int out_location, uint64_t* slow_alloc) {
  using namespace remap;
  if (H > 0x7FFFFFFFULL)  // remap.cpp:42-46
    throw InvalidArgument("table " + std::to_string(table_id) + ": hash_size " +
                          std::to_string(H) +
                          " exceeds the 2^31-1 limit of the signed 32-bit remap encoding");
  if (hbm_rows > H)  // remap.cpp:47-51
    throw InvalidArgument("table " + std::to_string(table_id) + ": hbm_rows " +
                          std::to_string(hbm_rows) + " exceeds hash_size " + std::to_string(H));
  if (distinct > H)
    throw InvalidArgument("table " + std::to_string(table_id) +
                          ": stats rank more rows than hash_size");
  if (distinct > 0 && rows_by_rank == nullptr)  // remap.cpp:52-56
    throw InvalidArgument("table " + std::to_string(table_id) +
                          ": stats lack row-level ranking (loaded from a stats file?); "
                          "re-profile the trace");
  cudaStream_t st = ctx->stream;
  const uint64_t ranked_fast = hbm_rows < distinct ? hbm_rows : distinct;
  const uint64_t extra = hbm_rows > distinct ? hbm_rows - distinct : 0;
  Scratch scr = ctx->scratch(Scratch::bytes_for(H + 1, 4) * 2 + Scratch::bytes_for(H + 1, 8) +
                             scan_scratch_bytes(H + 1, 8) + Scratch::bytes_for(distinct + 1, 4) +
                             (4 << 20));
  uint32_t* m = scr.take<uint32_t>(H + 1);
  uint64_t* ord = scr.take<uint64_t>(H + 1);
  uint64_t* tot = scr.take<uint64_t>(1);
  unsigned* err = scr.take<unsigned>(1);
  const uint32_t* d_rbr = rows_location == RS_MEM_DEVICE
                              ? rows_by_rank
                              : stage(rows_by_rank, distinct, false, scr, st);
  int32_t* d_out = out_location == RS_MEM_DEVICE ? entries : scr.take<int32_t>(H + 1);
  RS_CUDA(cudaMemsetAsync(m, 0xFF, H * 4, st));
  RS_CUDA(cudaMemsetAsync(err, 0, 4, st));
  const unsigned g = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>((std::max(H, distinct) + 255) / 256, uint64_t(sm_count()) * 16)));
  if (distinct) scatter_ranks<<<g, 256, 0, st>>>(d_rbr, distinct, H, m, err);
  exclusive_scan<uint64_t>(ClassFlags{m, uint32_t(ranked_fast)}, H, ord, tot, scr, st);
  if (H)
    finalize<<<g, 256, 0, st>>>(m, ord, tot, H, uint32_t(ranked_fast), distinct, extra, omit != 0,
                                d_out);
  RS_LAUNCH_CHECK();
  auto* hb = ctx->pinned_buf<uint64_t>(2);
  RS_CUDA(cudaMemcpyAsync(hb, tot, 8, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaMemcpyAsync(hb + 1, err, 4, cudaMemcpyDeviceToHost, st));
  if (out_location != RS_MEM_DEVICE && H)
    RS_CUDA(cudaMemcpyAsync(entries, d_out, H * 4, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  if (uint32_t(hb[1])) throw InvalidArgument("build_remap: rows_by_rank entry >= hash_size");
  const uint64_t nB = hb[0] >> 32, nC = hb[0] & 0xFFFFFFFFull;
  if (slow_alloc) *slow_alloc = omit ? nB : (nB + nC - extra);  // remap.cpp:92 / :102
}

}  // namespace rs

// ------------------------------------------------------------------ SPRM files
// The reference's binary remap format (core/src/remap.cpp:118-176): "SPRM",
// version 1, table_id u64, hash_size u64, hbm_rows u64 (little endian), then
// hash_size int32 entries (little endian — the in-memory layout on the GPU's
// hosts).  Reading streams the entries through a pinned buffer straight into
// device memory in chunks (DMA overlapping the file read); the slow-row count
// the reference recomputes on load is a device reduction.
#include <cstdio>
#include <cstring>

namespace rs {
namespace remap {

constexpr size_t kSprmHeader = 29;  // RemapTable::kHeaderBytes

__global__ void count_negative(const int32_t* __restrict__ e, uint64_t n, unsigned long long* __restrict__ out) {
  uint64_t c = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    c += e[i] < 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

}  // namespace remap

static void put_u64(unsigned char* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = (v >> (8 * i)) & 0xFF;
}
static uint64_t get_u64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
  return v;
}

void remap_write(rs_context* ctx, const char* path, uint32_t table_id, uint64_t H, uint64_t hbm_rows,
                 const int32_t* entries, int location) {
  FILE* f = std::fopen(path, "wb");
  if (!f) throw IoError(std::string("cannot open for writing: ") + path);
  unsigned char header[remap::kSprmHeader];
  std::memcpy(header, "SPRM", 4);
  header[4] = 1;
  put_u64(header + 5, table_id);
  put_u64(header + 13, H);
  put_u64(header + 21, hbm_rows);
  bool ok = std::fwrite(header, 1, sizeof header, f) == sizeof header;
  if (location == RS_MEM_DEVICE) {
    constexpr size_t kChunk = size_t(16) << 20;  // entries per DMA chunk
    int32_t* hb = ctx->pinned_buf<int32_t>(std::min<uint64_t>(H, kChunk));
    for (uint64_t i = 0; ok && i < H; i += kChunk) {
      const size_t n = size_t(std::min<uint64_t>(kChunk, H - i));
      RS_CUDA(cudaMemcpyAsync(hb, entries + i, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      ok = std::fwrite(hb, 4, n, f) == n;
    }
  } else if (H) {
    ok = ok && std::fwrite(entries, 4, H, f) == H;
  }
  if (std::fclose(f) != 0 || !ok) throw IoError(std::string("write failed: ") + path);
}

// Header only (table_id, hash_size, hbm_rows) — sizes the caller's buffer.
void remap_read_header(const char* path, uint32_t* table_id, uint64_t* H, uint64_t* hbm_rows) {
  FILE* f = std::fopen(path, "rb");
  if (!f) throw IoError(std::string("cannot open: ") + path);
  unsigned char header[remap::kSprmHeader];
  const bool got = std::fread(header, 1, sizeof header, f) == sizeof header;
  std::fclose(f);
  if (!got) throw ParseError(std::string("remap file too short: ") + path);
  if (std::memcmp(header, "SPRM", 4) != 0 || header[4] != 1)
    throw ParseError(std::string("bad remap magic or version: ") + path);
  *table_id = uint32_t(get_u64(header + 5));
  *H = get_u64(header + 13);
  *hbm_rows = get_u64(header + 21);
  if (*H > 0x7FFFFFFFULL) throw ParseError(std::string("remap hash_size out of range: ") + path);
}

void remap_read(rs_context* ctx, const char* path, int32_t* out, int location, uint64_t capacity,
                uint64_t* slow_rows_allocated) {
  uint32_t tid;
  uint64_t H, hbm;
  remap_read_header(path, &tid, &H, &hbm);
  if (H > capacity) throw InvalidArgument("read_remap: output buffer smaller than hash_size");
  FILE* f = std::fopen(path, "rb");
  if (!f) throw IoError(std::string("cannot open: ") + path);
  std::fseek(f, long(remap::kSprmHeader), SEEK_SET);
  uint64_t slow = 0;
  bool ok = true;
  if (location == RS_MEM_DEVICE) {
    cudaStream_t st = ctx->stream;
    // double-buffered: read chunk k+1 from the file while chunk k is on the bus
    constexpr size_t kChunk = size_t(8) << 20;
    int32_t* hb = ctx->pinned_buf<int32_t>(2 * std::min<uint64_t>(std::max<uint64_t>(H, 1), kChunk));
    const size_t cap = size_t(std::min<uint64_t>(std::max<uint64_t>(H, 1), kChunk));
    cudaEvent_t done[2];
    RS_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    RS_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    int k = 0;
    for (uint64_t i = 0; ok && i < H; i += cap, k ^= 1) {
      const size_t n = size_t(std::min<uint64_t>(cap, H - i));
      if (i >= 2 * cap) RS_CUDA(cudaEventSynchronize(done[k]));
      ok = std::fread(hb + k * cap, 4, n, f) == n;
      if (ok) {
        RS_CUDA(cudaMemcpyAsync(out + i, hb + k * cap, n * 4, cudaMemcpyHostToDevice, st));
        RS_CUDA(cudaEventRecord(done[k], st));
      }
    }
    Scratch scr = ctx->scratch(4096);
    auto* d_slow = scr.take<unsigned long long>(1);
    RS_CUDA(cudaMemsetAsync(d_slow, 0, 8, st));
    if (ok && H) {
      const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((H + 255) / 256, uint64_t(sm_count()) * 8)));
      remap::count_negative<<<g, 256, 0, st>>>(out, H, d_slow);
      RS_COUNT(1);
      RS_LAUNCH_CHECK();
    }
    unsigned long long hs = 0;
    RS_CUDA(cudaMemcpyAsync(&hs, d_slow, 8, cudaMemcpyDeviceToHost, st));
    ctx->sync();
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
    slow = hs;
  } else {
    ok = std::fread(out, 4, H, f) == H;
    for (uint64_t i = 0; ok && i < H; ++i) slow += out[i] < 0;
  }
  std::fclose(f);
  if (!ok) throw ParseError(std::string("remap file truncated: ") + path);
  if (slow_rows_allocated) *slow_rows_allocated = slow;
}

}  // namespace rs
