// HBM staging of slow-tier (UVM) rows, overlapped with compute (included by
// emb.cu).
//
// The plan leaves rows in pinned host memory that the GPU reads zero-copy over
// PCIe; inside the forward/backward those reads sit on the critical path.
// With a prefetch, each batch's slow rows are copied once (deduplicated) into
// an HBM staging area on a side stream BEFORE the batch runs — while the
// previous batch computes — the forward/backward read and update the staged
// copy, and a write-back on the side stream returns updated rows to the host
// tier while the next batch computes.  Values and arithmetic are unchanged
// (the staged row is the host row), so results are bit-identical to the
// zero-copy path; accounting (tier hits) still follows the remap.
//
// Per slow row: slot_of[s] = staging slot or kNoSlot.  Per slot: its (table,
// slow row) and a 2-bit generation mask — bit (g & 1) is set while batch g
// needs the row.  Two batches may be live (current + prefetched): a gather
// marks rows already staged instead of re-reading them (so a row updated by
// the running backward is never read stale from the host), and the write-back
// of batch g keeps rows batch g+1 still needs.  Gathers and write-backs run on
// one side stream, so slot allocation and release never race.
#pragma once

namespace rs {
namespace emb {

constexpr uint32_t kNoSlot = 0xFFFFFFFFu;
constexpr uint32_t kClaim = 0xFFFFFFFEu;

// Claim / mark the staging slots of one batch's slow rows.  New slots are
// queued in copy_list for the copy kernel.
__global__ void __launch_bounds__(256)
uvm_claim_kernel(const TableDev* __restrict__ tables, uint32_t T, uint64_t B,
                 const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ indices,
                 uint32_t gen_bit, uint32_t* __restrict__ slot_gen, uint32_t* __restrict__ slot_tab,
                 uint32_t* __restrict__ slot_row, uint32_t* __restrict__ free_stack,
                 int* __restrict__ free_top, uint32_t* __restrict__ copy_list,
                 unsigned* __restrict__ ncopy, unsigned* __restrict__ err) {
  const uint64_t nbags = uint64_t(T) * B;
  const uint64_t L = offsets[nbags];
  for (uint64_t l = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; l < L;
       l += uint64_t(gridDim.x) * blockDim.x) {
    // table of lookup l: tables are contiguous ranges of the CSR
    uint32_t lo = 0, hi = T;
    while (lo + 1 < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (offsets[uint64_t(mid) * B] <= l) lo = mid;
      else hi = mid;
    }
    while (lo + 1 < T && offsets[uint64_t(lo + 1) * B] <= l) ++lo;
    const TableDev& td = tables[lo];
    const int32_t e = td.remap[indices[l]];
    if (e >= 0) continue;
    const uint32_t s = uint32_t(-int64_t(e) - 1);
    uint32_t* p = td.slot_of + s;
    const uint32_t old = atomicCAS(p, kNoSlot, kClaim);
    if (old == kNoSlot) {
      const int top = atomicSub(free_top, 1);
      if (top <= 0) {
        atomicOr(err, 1u);
        atomicAdd(free_top, 1);
        atomicExch(p, kNoSlot);
        continue;
      }
      const uint32_t slot = free_stack[top - 1];
      slot_tab[slot] = lo;
      slot_row[slot] = s;
      slot_gen[slot] = gen_bit;
      copy_list[atomicAdd(ncopy, 1u)] = slot;
      __threadfence();
      atomicExch(p, slot);
    } else if (old != kClaim) {
      atomicOr(&slot_gen[old], gen_bit);
    }
  }
}

// Host row -> staging slot, one warp per newly claimed slot.
__global__ void __launch_bounds__(256)
uvm_fill_kernel(const TableDev* __restrict__ tables, const uint32_t* __restrict__ slot_tab,
                const uint32_t* __restrict__ slot_row, const uint32_t* __restrict__ copy_list,
                const unsigned* __restrict__ ncopy, float* __restrict__ staging, uint64_t stride) {
  const int lane = threadIdx.x & 31;
  const uint64_t n = *ncopy;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
    const uint32_t slot = copy_list[i];
    const TableDev& td = tables[slot_tab[slot]];
    const float4* src = reinterpret_cast<const float4*>(td.slow + uint64_t(slot_row[slot]) * td.dim);
    float4* dst = reinterpret_cast<float4*>(staging + uint64_t(slot) * stride);
    for (uint32_t v = lane; v < (td.dim >> 2); v += 32) dst[v] = src[v];
  }
}

// Release every slot of generation bit `gen_bit` that no batch in `keep`
// still needs: staged row -> host row, slot_of reset, slot back on the free
// stack.  Rows kept for the next batch only lose the bit.
__global__ void __launch_bounds__(256)
uvm_writeback_kernel(const TableDev* __restrict__ tables, uint32_t nslots, uint32_t gen_bit,
                     uint32_t keep, uint32_t* __restrict__ slot_gen, const uint32_t* __restrict__ slot_tab,
                     const uint32_t* __restrict__ slot_row, uint32_t* __restrict__ free_stack,
                     int* __restrict__ free_top, const float* __restrict__ staging, uint64_t stride) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t base = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; base < nslots;
       base += nwarps * 32) {
    const uint32_t my = uint32_t(base) + lane;
    const uint32_t g = my < nslots ? slot_gen[my] : 0u;
    const bool mine = (g & gen_bit) != 0;
    const bool kept = mine && (g & keep) != 0;
    if (kept) slot_gen[my] = g & ~gen_bit;
    unsigned evict = __ballot_sync(0xffffffffu, mine && !kept);
    while (evict) {
      const int src = __ffs(evict) - 1;
      evict &= evict - 1;
      const uint32_t slot = uint32_t(base) + src;
      const TableDev& td = tables[slot_tab[slot]];
      const uint32_t s = slot_row[slot];
      const float4* from = reinterpret_cast<const float4*>(staging + uint64_t(slot) * stride);
      float4* to = reinterpret_cast<float4*>(td.slow + uint64_t(s) * td.dim);
      for (uint32_t v = lane; v < (td.dim >> 2); v += 32) to[v] = from[v];
      if (lane == 0) {
        td.slot_of[s] = kNoSlot;
        slot_gen[slot] = 0;
        free_stack[atomicAdd(free_top, 1)] = slot;
      }
    }
  }
}

}  // namespace emb
}  // namespace rs
