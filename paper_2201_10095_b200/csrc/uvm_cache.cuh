// HBM staging of slow-tier (UVM) rows, moved by the copy engines while the
// previous batch computes (included by emb.cu).
//
// The plan leaves rows in pinned host memory that the kernels could read
// zero-copy over PCIe — but SM-issued PCIe traffic costs about its own
// duration in lost HBM throughput (measured: a concurrent zero-copy gather
// slowed the backward by ~1 ms, a concurrent DMA of the same bytes by 0.1 ms).
// So each batch's slow rows are staged once (deduplicated) into HBM slots
// BEFORE the batch runs: a claim kernel (caller's stream) lists the rows that
// are not staged yet, a host worker gathers them from the host tier into a
// pinned bounce buffer (CPU memcpy, several threads) and one DMA copy plus a
// scatter kernel put them in their slots (side stream).  After the backward,
// an evict kernel (caller's stream) packs the rows no pending batch needs
// into a device bounce buffer and frees their slots; the worker copies them
// back with one DMA and scatters them into the host tier.  Values and
// arithmetic are unchanged (a staged row IS the host row), so results are
// bit-identical to the zero-copy path; accounting follows the remap.
//
// Per slow row: slot_of[s] = staging slot or kNoSlot.  Per slot: its (table,
// slow row) and a 2-bit generation mask — bit (g & 1) is set while batch g
// needs the row.  Two batches may be live (current + prefetched): a claim
// marks rows already staged instead of re-reading them (so a row updated by
// the running backward is never read stale from the host), and the eviction
// of batch g keeps rows batch g+1 still needs.  Claims and evictions run on
// the caller's stream, so slot allocation and release never race; the host
// worker runs its gathers and scatters in FIFO order, so a row evicted by
// batch g reaches the host tier before a later batch gathers it again.
#pragma once

namespace rs {
namespace emb {

constexpr uint32_t kNoSlot = 0xFFFFFFFFu;
constexpr uint32_t kClaim = 0xFFFFFFFEu;
constexpr uint32_t kDeadRow = 0xFFFFFFFFu;  // slot_row of a slot whose copy-list entry overflowed

// A warp copies one row of `bytes` (a multiple of 8: dim % 4 == 0 rows of
// fp32 or fp16), 16 bytes per lane-access when the row allows it.
__device__ __forceinline__ void copy_row_bytes(char* dst, const char* src, uint32_t bytes, int lane) {
  if ((bytes & 15) == 0) {
    for (uint32_t v = lane; v < bytes / 16; v += 32)
      reinterpret_cast<float4*>(dst)[v] = reinterpret_cast<const float4*>(src)[v];
  } else {
    for (uint32_t v = lane; v < bytes / 8; v += 32)
      reinterpret_cast<uint2*>(dst)[v] = reinterpret_cast<const uint2*>(src)[v];
  }
}

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
                 uint32_t* __restrict__ copy_tab, uint32_t* __restrict__ copy_row, uint32_t cap,
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
      const uint32_t r = indices[l];
      if (!((td.sbits[r >> 5] >> (r & 31)) & 1u)) continue;  // fast or unbacked: nothing to stage
      const int32_t e = td.remap[r];
      const uint64_t s = slow_off(e);
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
        slot_row[slot] = uint32_t(s);
        slot_gen[slot] = gen_bit;
        const unsigned k = atomicAdd(ncopy, 1u);
        if (k < cap) {
          copy_list[k] = slot;
          copy_tab[k] = t;
          copy_row[k] = uint32_t(s);
          __threadfence();
          atomicExch(p, slot);
        } else {
          // no room to copy the row in: the slot is never filled, so the row
          // keeps no slot (row_ptr falls back to the host tier) and the slot
          // is freed by the next eviction without a write-back
          slot_row[slot] = kDeadRow;
          atomicOr(err, 2u);
          __threadfence();
          atomicExch(p, kNoSlot);
        }
      } else if (old != kClaim) {
        atomicOr(&slot_gen[old], gen_bit);
      }
    }
  }
}

// Bounce row k (the host row, copied by DMA) -> its staging slot; warp per row.
__global__ void __launch_bounds__(256)
uvm_scatter_in_kernel(const TableDev* __restrict__ tables, const uint32_t* __restrict__ copy_list,
                      const uint32_t* __restrict__ copy_tab, const unsigned* __restrict__ ncopy, uint32_t cap,
                      const char* __restrict__ bounce, char* __restrict__ staging, uint64_t stride) {
  const int lane = threadIdx.x & 31;
  const uint64_t n = min(*ncopy, cap);
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t k = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; k < n; k += nwarps)
    copy_row_bytes(staging + uint64_t(copy_list[k]) * stride, bounce + k * stride, tables[copy_tab[k]].rbytes, lane);
}

// Release every slot of generation bit `gen_bit` that no batch in `keep`
// still needs: staged row -> bounce row k (with its table / slow row for the
// host scatter), slot_of reset, slot back on the free stack.  Rows kept for
// the next batch only lose the bit.
__global__ void __launch_bounds__(256)
uvm_evict_kernel(const TableDev* __restrict__ tables, uint32_t nslots, uint32_t gen_bit, uint32_t keep,
                 uint32_t* __restrict__ slot_gen, const uint32_t* __restrict__ slot_tab,
                 const uint32_t* __restrict__ slot_row, uint32_t* __restrict__ free_stack,
                 int* __restrict__ free_top, const char* __restrict__ staging, uint64_t stride,
                 char* __restrict__ bounce, uint32_t* __restrict__ wb_tab, uint32_t* __restrict__ wb_row,
                 uint32_t cap, unsigned* __restrict__ n_wb, unsigned* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t base = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; base < nslots;
       base += nwarps * 32) {
    const uint32_t my = uint32_t(base) + lane;
    const uint32_t g = my < nslots ? slot_gen[my] : 0u;
    const bool mine = (g & gen_bit) != 0;
    const bool kept = mine && (g & keep) != 0;
    if (kept) slot_gen[my] = g & ~gen_bit;
    // a slot whose row was never copied in (kDeadRow) is freed without a write-back
    const bool dead = mine && !kept && slot_row[my] == kDeadRow;
    if (dead) {
      slot_gen[my] = 0;
      free_stack[atomicAdd(free_top, 1)] = my;
    }
    unsigned evict = __ballot_sync(0xffffffffu, mine && !kept && !dead);
    unsigned k0 = 0;
    if (lane == 0 && evict) k0 = atomicAdd(n_wb, unsigned(__popc(evict)));
    k0 = __shfl_sync(0xffffffffu, k0, 0);
    while (evict) {
      const int src = __ffs(evict) - 1;
      evict &= evict - 1;
      const uint32_t slot = uint32_t(base) + src;
      const uint32_t t = slot_tab[slot];
      const TableDev& td = tables[t];
      const uint32_t s = slot_row[slot];
      if (k0 < cap) {
        copy_row_bytes(bounce + uint64_t(k0) * stride, staging + uint64_t(slot) * stride, td.rbytes, lane);
        if (lane == 0) {
          wb_tab[k0] = t;
          wb_row[k0] = s;
        }
      } else if (lane == 0) {
        atomicOr(err, 2u);
      }
      if (lane == 0) {
        td.slot_of[s] = kNoSlot;
        slot_gen[slot] = 0;
        free_stack[atomicAdd(free_top, 1)] = slot;
      }
      ++k0;
    }
  }
}

}  // namespace emb
}  // namespace rs
