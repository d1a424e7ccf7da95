// HP2 accounting — simulate() on the GPU (core/src/simulator.cpp:26-139).
//
// The hot loop (:80-94) becomes one pass over the trace: every record of a
// full batch (sample < batches*B) routes its ids through its table's remap and
// counts fast (entry >= 0) hits.  The GPU produces exact per-table u64
// (fast, total) counts; the per-GPU counts follow by summing tables on the
// host, and the report formulas (:96-137) are applied on the host exactly as
// the reference writes them.  Each reference partial sum double(fast)*row_bytes
// is an integer < 2^53, so the double sums are order-independent: bit-exact.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <unordered_map>

#include "../../include/shardplan_gpu.h"
#include "context.cuh"

namespace rs {
namespace sim {

constexpr int kThreads = 256;
constexpr uint32_t kMaxSmemTables = 2048;

__device__ __forceinline__ int lookup(const uint32_t* __restrict__ sid, const uint32_t* __restrict__ six,
                                      uint32_t J, uint32_t id) {
  uint32_t lo = 0, hi = J;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (sid[mid] < id) lo = mid + 1;
    else hi = mid;
  }
  return (lo < J && sid[lo] == id) ? int(six[lo]) : -1;
}

__global__ void __launch_bounds__(kThreads)
tier_counts(const uint64_t* __restrict__ rec_sample, const uint32_t* __restrict__ rec_table,
            const uint64_t* __restrict__ rec_offset, const uint32_t* __restrict__ rec_len, uint64_t R,
            const uint32_t* __restrict__ ids, uint64_t sample_limit, const uint32_t* __restrict__ sid,
            const uint32_t* __restrict__ six, uint32_t J, const uint64_t* __restrict__ rbase,
            const uint64_t* __restrict__ hsize, const int32_t* __restrict__ remap,
            unsigned long long* __restrict__ fast_out, unsigned long long* __restrict__ total_out,
            unsigned* __restrict__ err) {
  extern __shared__ unsigned long long smc[];
  const bool use_sm = J <= kMaxSmemTables;
  if (use_sm)
    for (uint32_t i = threadIdx.x; i < 2 * J; i += blockDim.x) smc[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t c = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c * 32 < R; c += nwarps) {
    const uint64_t r = c * 32 + lane;
    uint32_t len = 0;
    uint64_t off = 0;
    int t = 0;
    if (r < R && rec_sample[r] < sample_limit) {  // simulator.cpp:81
      t = lookup(sid, six, J, rec_table[r]);
      if (t < 0) {
        atomicOr(err, 1u);
        t = 0;
      } else {
        len = rec_len[r];
        off = rec_offset[r];
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
        uint32_t e = __shfl_sync(0xffffffffu, excl, k + step);
        if (e <= q) k += step;
      }
      const uint64_t offk = __shfl_sync(0xffffffffu, off, k);
      const uint32_t exk = __shfl_sync(0xffffffffu, excl, k);
      const int tk = __shfl_sync(0xffffffffu, t, k);
      const unsigned act = __ballot_sync(0xffffffffu, q < total);
      if (q < total) {
        const uint32_t row = ld_stream_u32(ids + offk + (q - exk));
        bool fast = false;
        if (row >= hsize[tk]) atomicOr(err, 2u);
        else fast = remap[rbase[tk] + row] >= 0;  // simulator.cpp:86
        // warp-aggregate per table: peers share (table, fast) in this round
        const unsigned peers = __match_any_sync(act, tk);
        const unsigned fm = __ballot_sync(act, fast) & peers;
        if ((peers & lanemask_lt()) == 0) {
          if (use_sm) {
            atomicAdd(&smc[2 * tk], (unsigned long long)__popc(fm));
            atomicAdd(&smc[2 * tk + 1], (unsigned long long)__popc(peers));
          } else {
            atomicAdd(&fast_out[tk], (unsigned long long)__popc(fm));
            atomicAdd(&total_out[tk], (unsigned long long)__popc(peers));
          }
        }
      }
    }
  }
  if (use_sm) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < J; i += blockDim.x) {
      if (smc[2 * i + 1]) {
        atomicAdd(&fast_out[i], smc[2 * i]);
        atomicAdd(&total_out[i], smc[2 * i + 1]);
      }
    }
  }
}

}  // namespace sim

void simulate(rs_context* ctx, const rs_trace* tr, uint32_t ne, const rs_plan_entry* entries,
              uint32_t nr, const rs_remap_view* remaps, const rs_system_spec* sys,
              uint64_t batch_size, rs_sim_report* out) {
  using namespace sim;
  // validate(system), types.hpp:97-108
  if (sys->num_gpus < 1) throw InvalidArgument("system: num_gpus must be >= 1");
  if (sys->batch_size < 1) throw InvalidArgument("system: batch_size must be >= 1");
  if (sys->cap_hbm_bytes < 1) throw InvalidArgument("system: cap_hbm_bytes must be positive");
  if (sys->cap_dram_bytes < 1) throw InvalidArgument("system: cap_dram_bytes must be positive");
  if (!(sys->bw_hbm > 0.0) || !(sys->bw_uvm > 0.0))
    throw InvalidArgument("system: bandwidths must be positive");
  if (!(sys->bw_hbm > sys->bw_uvm)) throw InvalidArgument("system: bw_hbm must exceed bw_uvm");
  if (batch_size < 1) throw InvalidArgument("simulate: batch_size must be >= 1");  // :30
  const uint64_t batches = tr->num_samples / batch_size;                          // :31-34
  if (batches == 0) throw InvalidArgument("simulate: trace holds fewer samples than one batch");
  if (!tr->ids) throw InvalidArgument("simulate: trace must carry hashed ids");

  // :36-70 routing tables, validated in trace table order
  std::unordered_map<uint32_t, const rs_plan_entry*> entry_of;
  for (uint32_t i = 0; i < ne; ++i) entry_of[entries[i].table_id] = &entries[i];
  std::unordered_map<uint32_t, const rs_remap_view*> remap_of;
  for (uint32_t i = 0; i < nr; ++i) remap_of[remaps[i].table_id] = &remaps[i];
  const uint32_t J = tr->num_tables;
  std::vector<uint32_t> gpu(J);
  std::vector<const rs_remap_view*> rv(J);
  std::vector<double> row_bytes(J);
  for (uint32_t j = 0; j < J; ++j) {
    const rs_table_spec& t = tr->tables[j];
    auto eit = entry_of.find(t.table_id);
    if (eit == entry_of.end())
      throw InvalidArgument("simulate: trace table " + std::to_string(t.table_id) +
                            " missing from plan");
    auto rit = remap_of.find(t.table_id);
    if (rit == remap_of.end())
      throw InvalidArgument("simulate: no remap for table " + std::to_string(t.table_id));
    if (rit->second->hash_size != t.hash_size)
      throw InvalidArgument("simulate: remap for table " + std::to_string(t.table_id) + " sized " +
                            std::to_string(rit->second->hash_size) + ", trace says " +
                            std::to_string(t.hash_size));
    if (eit->second->gpu >= sys->num_gpus)
      throw InvalidArgument("simulate: table " + std::to_string(t.table_id) +
                            " assigned to gpu " + std::to_string(eit->second->gpu) +
                            " outside system");
    gpu[j] = eit->second->gpu;
    rv[j] = rit->second;
    row_bytes[j] = static_cast<double>(t.dim) * t.elem_bytes;
  }

  cudaStream_t st = ctx->stream;
  const bool on_dev = tr->location == RS_MEM_DEVICE;
  const uint64_t R = tr->num_records, N = tr->num_ids;
  std::vector<uint64_t> rbase(J + 1, 0), hs(J);
  for (uint32_t j = 0; j < J; ++j) {
    hs[j] = tr->tables[j].hash_size;
    rbase[j + 1] = rbase[j] + hs[j];
  }
  Scratch scr = ctx->scratch(Scratch::bytes_for(R, 8) * 2 + Scratch::bytes_for(R, 4) * 2 +
                             Scratch::bytes_for(N, 4) + Scratch::bytes_for(rbase[J] + 1, 4) +
                             Scratch::bytes_for(J + 1, 8) * 8 + (4 << 20));
  const uint64_t* d_rs = on_dev ? tr->rec_sample : stage(tr->rec_sample, R, false, scr, st);
  const uint32_t* d_rt = on_dev ? tr->rec_table : stage(tr->rec_table, R, false, scr, st);
  const uint64_t* d_ro = on_dev ? tr->rec_offset : stage(tr->rec_offset, R, false, scr, st);
  const uint32_t* d_rl = on_dev ? tr->rec_len : stage(tr->rec_len, R, false, scr, st);
  const uint32_t* d_ids = on_dev ? tr->ids : stage(tr->ids, N, false, scr, st);
  int32_t* d_remap = scr.take<int32_t>(rbase[J] + 1);
  for (uint32_t j = 0; j < J; ++j)
    if (hs[j])
      RS_CUDA(cudaMemcpyAsync(d_remap + rbase[j], rv[j]->entries, hs[j] * 4,
                              rv[j]->location == RS_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                               : cudaMemcpyHostToDevice,
                              st));
  std::vector<uint32_t> order(J), sid(J), six(J);
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(),
            [&](uint32_t a, uint32_t b) { return tr->tables[a].table_id < tr->tables[b].table_id; });
  for (uint32_t i = 0; i < J; ++i) {
    sid[i] = tr->tables[order[i]].table_id;
    six[i] = order[i];
  }
  uint32_t* d_sid = stage(sid.data(), J, false, scr, st);
  uint32_t* d_six = stage(six.data(), J, false, scr, st);
  uint64_t* d_rbase = stage(rbase.data(), J + 1, false, scr, st);
  uint64_t* d_hs = stage(hs.data(), J, false, scr, st);
  auto* d_cnt = scr.take<unsigned long long>(2 * size_t(J));
  auto* d_err = scr.take<unsigned>(1);
  RS_CUDA(cudaMemsetAsync(d_cnt, 0, 2 * size_t(J) * 8, st));
  RS_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
  const uint64_t warps = (R + 31) / 32;
  unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, uint64_t(sm_count()) * 8)));
  size_t smem = J <= kMaxSmemTables ? size_t(J) * 16 : 0;
  tier_counts<<<grid, kThreads, smem, st>>>(d_rs, d_rt, d_ro, d_rl, R, d_ids, batches * batch_size,
                                            d_sid, d_six, J, d_rbase, d_hs, d_remap, d_cnt, d_cnt + J,
                                            d_err);
  RS_LAUNCH_CHECK();
  auto* hb = ctx->pinned_buf<uint64_t>(2 * size_t(J) + 1);
  RS_CUDA(cudaMemcpyAsync(hb, d_cnt, 2 * size_t(J) * 8, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaMemcpyAsync(hb + 2 * J, d_err, 4, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  if (uint32_t(hb[2 * J]) & 1u)
    throw OutOfRange("simulate: record references a table id absent from trace.tables");
  if (uint32_t(hb[2 * J]) & 2u) throw InvalidArgument("simulate: hashed id outside its table");

  // :96-137 — report from exact counts
  const uint32_t M = sys->num_gpus;
  std::vector<uint64_t> hbm(M, 0), uvm(M, 0);
  std::vector<double> hbm_b(M, 0.0), uvm_b(M, 0.0);
  for (uint32_t j = 0; j < J; ++j) {
    const uint64_t fast = hb[j], tot = hb[J + j];
    hbm[gpu[j]] += fast;
    uvm[gpu[j]] += tot - fast;
    hbm_b[gpu[j]] += static_cast<double>(fast) * row_bytes[j];
    uvm_b[gpu[j]] += static_cast<double>(tot - fast) * row_bytes[j];
  }
  out->batches = batches;
  uint64_t total_hbm = 0, total_uvm = 0;
  const double bi = static_cast<double>(batches);
  for (uint32_t g = 0; g < M; ++g) {
    out->gpu_hbm_accesses[g] = static_cast<double>(hbm[g]) / bi;
    out->gpu_uvm_accesses[g] = static_cast<double>(uvm[g]) / bi;
    out->gpu_est_iter_cost[g] = (hbm_b[g] / sys->bw_hbm + uvm_b[g] / sys->bw_uvm) / bi;
    total_hbm += hbm[g];
    total_uvm += uvm[g];
  }
  out->total_accesses = total_hbm + total_uvm;
  out->uvm_access_fraction =
      out->total_accesses ? static_cast<double>(total_uvm) / out->total_accesses : 0.0;
  double mn = std::numeric_limits<double>::max(), mx = 0.0, sum = 0.0;
  for (uint32_t g = 0; g < M; ++g) {
    mn = std::min(mn, out->gpu_est_iter_cost[g]);
    mx = std::max(mx, out->gpu_est_iter_cost[g]);
    sum += out->gpu_est_iter_cost[g];
  }
  out->min_cost = mn;
  out->max_cost = mx;
  out->mean_cost = sum / M;
  double var = 0.0;
  for (uint32_t g = 0; g < M; ++g) {
    double d = out->gpu_est_iter_cost[g] - out->mean_cost;
    var += d * d;
  }
  out->stddev_cost = std::sqrt(var / M);
  for (uint32_t j = 0; j < J; ++j)
    out->table_fast_fraction[j] = hb[J + j] ? static_cast<double>(hb[j]) / hb[J + j]
                                            : std::numeric_limits<double>::quiet_NaN();
}

}  // namespace rs
