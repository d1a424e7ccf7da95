// Shared between the operator (emb.cu) and the rank exchange (exchange.cu):
// the forward's output map and the few operator fields the exchange drives.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

struct rs_emb;
struct rs_context;

namespace rs {

constexpr int kMaxRanks = 8;  // one NVSwitch node

// Where bag (t, b)'s pooled row goes.  Local: the caller's [B, stride]
// output at the table's operator column td.col.  Exchange (K6 fused into
// K4): sample b's row is written straight into its owner's [bl, stride]
// block — peer memory over NVLink when the owner is another GPU — at the
// table's column in the GLOBAL table order, xcol[t].
struct OutMap {
  float* out0;               // n == 1: the [B, stride] output
  float* const* peers;       // n > 1: device array of each destination's block
  const uint32_t* xcol;      // [T] global columns (exchange) or nullptr (td.col)
  uint64_t bl;               // samples per destination rank
  uint32_t n;                // destination ranks
};

__device__ __forceinline__ float* out_row(const OutMap& om, uint64_t b, uint64_t stride) {
  if (om.n == 1) return om.out0 + b * stride;
  const uint64_t r = b / om.bl;
  return om.peers[r] + (b - r * om.bl) * stride;
}

void emb_forward_map(rs_emb* e, uint64_t B, const uint32_t* off, const uint32_t* idx, const OutMap& om,
                     uint64_t stride, uint64_t* hits);
void emb_backward(rs_emb* e, uint64_t B, const uint32_t* off, const uint32_t* idx, const float* grad, float lr);
// operator facts the exchange checks against its table map
uint32_t emb_num_tables(const rs_emb* e);
uint32_t emb_table_id(const rs_emb* e, uint32_t t);
uint32_t emb_table_dim(const rs_emb* e, uint32_t t);
rs_context* emb_context(const rs_emb* e);
// the next backward waits for `ev` before it reads gradient rows
void emb_set_grad_ready(rs_emb* e, cudaEvent_t ev);

}  // namespace rs
