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
// queued in copy_list for the copy kernel.  Only tables with slow rows are
// walked; a warp takes 32 consecutive bags of one table and flattens their
// lookups (one per lane, coalesced index reads, no per-lookup table search).
__global__ void __launch_bounds__(256)
uvm_claim_kernel(const TableDev* __restrict__ tables, const uint32_t* __restrict__ slow_tabs,
                 uint32_t nslow, uint64_t B, const uint32_t* __restrict__ offsets,
                 const uint32_t* __restrict__ indices, uint32_t gen_bit,
                 uint32_t* __restrict__ slot_gen, uint32_t* __restrict__ slot_tab,
                 uint32_t* __restrict__ slot_row, uint32_t* __restrict__ free_stack,
                 int* __restrict__ free_top, uint32_t* __restrict__ copy_list,
                 unsigned* __restrict__ ncopy, unsigned* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const uint64_t cpt = (B + 31) / 32;  // 32-bag chunks per table
  const uint64_t nwork = uint64_t(nslow) * cpt;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t c = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < nwork; c += nwarps) {
    const uint32_t t = slow_tabs[c / cpt];
    const uint64_t b0 = (c % cpt) * 32;
    const uint64_t nb = min(uint64_t(32), B - b0);
    const uint64_t o = uint64_t(t) * B + b0;
    const uint32_t s0 = offsets[o];
    const uint32_t s1 = offsets[o + nb];
    const TableDev& td = tables[t];
    for (uint32_t l = s0 + lane; l < s1; l += 32) {
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
        slot_tab[slot] = t;
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
}

// Host row -> staging slot.  A warp copies RPW rows at a time (their PCIe
// reads all in flight before the HBM stores), so a small grid keeps the bus
// busy without holding many SM slots away from the compute stream.
constexpr int kFillRows = 8;
__global__ void __launch_bounds__(256)
uvm_fill_kernel(const TableDev* __restrict__ tables, const uint32_t* __restrict__ slot_tab,
                const uint32_t* __restrict__ slot_row, const uint32_t* __restrict__ copy_list,
                const unsigned* __restrict__ ncopy, float* __restrict__ staging, uint64_t stride) {
  const int lane = threadIdx.x & 31;
  const uint64_t n = *ncopy;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i0 = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kFillRows; i0 < n;
       i0 += nwarps * kFillRows) {
    uint32_t slot[kFillRows], V[kFillRows];
    const float4* src[kFillRows];
#pragma unroll
    for (int r = 0; r < kFillRows; ++r) {
      slot[r] = i0 + r < n ? copy_list[i0 + r] : 0u;
      V[r] = 0;
      src[r] = nullptr;
      if (i0 + r < n) {
        const TableDev& td = tables[slot_tab[slot[r]]];
        V[r] = td.dim >> 2;
        src[r] = reinterpret_cast<const float4*>(td.slow + uint64_t(slot_row[slot[r]]) * td.dim);
      }
    }
    uint32_t vmax = 0;
#pragma unroll
    for (int r = 0; r < kFillRows; ++r) vmax = max(vmax, V[r]);
    for (uint32_t v = lane; v < vmax; v += 32) {
      float4 x[kFillRows];
#pragma unroll
      for (int r = 0; r < kFillRows; ++r)
        if (v < V[r]) x[r] = src[r][v];
#pragma unroll
      for (int r = 0; r < kFillRows; ++r)
        if (v < V[r]) reinterpret_cast<float4*>(staging + uint64_t(slot[r]) * stride)[v] = x[r];
    }
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
