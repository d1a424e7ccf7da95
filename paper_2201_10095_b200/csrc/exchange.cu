// K6 — the pooled-row exchange of table-wise model parallelism (SURVEY §8e,
// §8b rs_emb_alltoall_{fwd,bwd}).
//
// Rank r owns the tables whose PlanEntry.gpu == r (both tiers on the owner,
// PAPER.md:550-552) and pools them for the WHOLE global batch B; rank r also
// owns samples [r*bl, (r+1)*bl), bl = B / N.  Forward: every sample owner
// needs its rows of every table, [bl, D_total] in the global table order;
// backward: every table owner needs its tables' gradient rows for all B
// samples, [B, D_local].  Two transports:
//
//  * RS_EX_PEER — NVLink peer memory (one process per GPU, buffers mapped with
//    CUDA IPC).  The forward is FUSED with K4: the gather-pool kernel stores
//    each bag's pooled row straight into its owner's block (peer stores ride
//    NVLink while the kernel computes; no send buffer, no pack), then a
//    system-scope flag barrier publishes the blocks.  The backward pulls the
//    gradient rows of this rank's tables out of every owner's block with one
//    peer-read kernel on a side stream, while K5's plan/sort/segment passes
//    (which need no gradient) run; K5's first gradient read waits for it.
//    Remote gradients are pulled ONCE into local memory rather than read in
//    K5's inner loop: K5 reads a bag's gradient row once per lookup, and
//    peer reads are not cached in the local L2.
//  * RS_EX_NCCL — grouped ncclSend/ncclRecv per peer on the operator's
//    streams (the baseline; also the cross-node transport).  K4 writes
//    [B, D_local] sample-major, which IS the destination-major send layout
//    (rows [s*bl, (s+1)*bl) go to rank s), so the forward sends without a
//    pack; the received source-major blocks are scattered into global
//    column order by one kernel.  The backward packs owner columns into
//    per-destination blocks with the same map and receives straight into
//    [B, D_local] (source r's block is rows [r*bl, (r+1)*bl)), overlapped
//    with K5's sort like the peer path.
//
// NCCL is resolved at run time (dlopen of the process's libnccl.so.2 — the
// one torch.distributed already loaded, if any), so the library does not
// link a second NCCL.
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/shardplan_gpu.h"
#include "context.cuh"
#include "exchange.cuh"

namespace rs {
namespace ex {

// ---------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static const Nccl& nccl() {
  static Nccl n;
  static bool done = false;
  if (done) return n;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw Error(RS_ERR_INTERNAL, std::string("exchange: cannot load libnccl.so.2: ") + dlerror());
  auto sym = [&](auto& f, const char* name) {
    f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
    if (!f) throw Error(RS_ERR_INTERNAL, std::string("exchange: libnccl.so.2 lacks ") + name);
  };
  sym(n.GetUniqueId, "ncclGetUniqueId");
  sym(n.CommInitRank, "ncclCommInitRank");
  sym(n.CommDestroy, "ncclCommDestroy");
  sym(n.GroupStart, "ncclGroupStart");
  sym(n.GroupEnd, "ncclGroupEnd");
  sym(n.Send, "ncclSend");
  sym(n.Recv, "ncclRecv");
  sym(n.GetErrorString, "ncclGetErrorString");
  done = true;
  return n;
}

#define RS_NCCL(expr)                                                                   \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess)                                                              \
      throw ::rs::Error(RS_ERR_INTERNAL, std::string(#expr) + ": " + ::rs::ex::nccl().GetErrorString(r_)); \
  } while (0)

// ---------------------------------------------------------------- kernels
// Column maps in float4 units.  gsrc/gcol: for each global column c of the
// owner layout [bl, D_total], the source rank and column within that rank's
// [.., D_rank] block.  lmap: for each local column of [B, D_local], its
// global column.

// NCCL forward: source-major received blocks -> [bl, D_total] global order.
__global__ void __launch_bounds__(256) assemble_kernel(const float4* __restrict__ recv,
                                                       const uint64_t* __restrict__ src_off4,
                                                       const uint32_t* __restrict__ src_d4,
                                                       const uint32_t* __restrict__ gsrc,
                                                       const uint32_t* __restrict__ gcol, uint64_t bl,
                                                       uint32_t D4, float4* __restrict__ out) {
  const uint64_t n = bl * D4;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t row = i / D4;
    const uint32_t c = uint32_t(i - row * D4);
    const uint32_t s = gsrc[c];
    out[i] = recv[src_off4[s] + row * src_d4[s] + gcol[c]];
  }
}

// NCCL backward: owner gradients [bl, D_total] -> per-destination blocks.
__global__ void __launch_bounds__(256) pack_kernel(const float4* __restrict__ grad_owned,
                                                   const uint64_t* __restrict__ dst_off4,
                                                   const uint32_t* __restrict__ dst_d4,
                                                   const uint32_t* __restrict__ gsrc,
                                                   const uint32_t* __restrict__ gcol, uint64_t bl, uint32_t D4,
                                                   float4* __restrict__ send) {
  const uint64_t n = bl * D4;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t row = i / D4;
    const uint32_t c = uint32_t(i - row * D4);
    const uint32_t s = gsrc[c];
    send[dst_off4[s] + row * dst_d4[s] + gcol[c]] = grad_owned[i];
  }
}

// Peer forward (the unfused primitive): [B, D_local] rows -> every owner's block.
__global__ void __launch_bounds__(256) push_kernel(const float4* __restrict__ local, float4* const* __restrict__ owners,
                                                   const uint32_t* __restrict__ lmap, uint64_t B, uint64_t bl,
                                                   uint32_t D4, uint32_t L4) {
  const uint64_t n = B * L4;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = i / L4;
    const uint32_t c = uint32_t(i - b * L4);
    const uint64_t r = b / bl;
    owners[r][(b - r * bl) * D4 + lmap[c]] = local[i];
  }
}

// Peer backward: this rank's columns of every owner's block -> [B, D_local].
__global__ void __launch_bounds__(256) pull_kernel(const float4* const* __restrict__ owners,
                                                   const uint32_t* __restrict__ lmap, uint64_t B, uint64_t bl,
                                                   uint32_t D4, uint32_t L4, float4* __restrict__ out,
                                                   const unsigned* __restrict__ err) {
  if (*reinterpret_cast<const volatile unsigned*>(err)) return;  // a peer never arrived
  const uint64_t n = B * L4;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = i / L4;
    const uint32_t c = uint32_t(i - b * L4);
    const uint64_t r = b / bl;
    out[i] = owners[r][(b - r * bl) * D4 + lmap[c]];
  }
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// All-rank barrier on flags in peer memory: thread s tells rank s that this
// rank reached `seq` (after everything earlier on the stream — its peer
// stores — is visible system-wide), then waits until rank s did the same.
// A peer that never arrives trips `err` after ~`spin_limit` polls instead of
// hanging the GPU.
__global__ void barrier_kernel(uint64_t* const* __restrict__ peer_flags, uint64_t* __restrict__ my_flags,
                               uint32_t me, uint32_t n, uint64_t seq, unsigned* __restrict__ err,
                               uint64_t spin_limit) {
  const uint32_t s = threadIdx.x;
  if (s >= n) return;
  __threadfence_system();
  st_release_sys(peer_flags[s] + me, seq);
  uint64_t spins = 0;
  while (ld_acquire_sys(my_flags + s) < seq) {
    __nanosleep(200);
    if (++spins > spin_limit) {
      atomicOr(err, 1u);
      break;
    }
  }
  __threadfence_system();
}

}  // namespace ex
}  // namespace rs

// The exchange handle: one per rank, bound to an operator's table set.
struct rs_exchange {
  rs_context* ctx = nullptr;
  int kind = RS_EX_PEER;
  uint32_t N = 1, rank = 0;
  uint64_t B = 0, bl = 0;
  uint32_t J = 0;                   // global tables
  std::vector<uint32_t> dims, owner, gcol;  // per global table
  std::vector<uint32_t> local;      // global indices owned here, ascending
  std::vector<uint32_t> xcol_h;     // global column of each local table
  std::vector<uint32_t> Drank;      // sum of dims per rank
  uint64_t D_total = 0, D_local = 0;
  // device maps
  uint32_t *gsrc = nullptr, *gcol4 = nullptr, *lmap = nullptr, *xcol = nullptr, *src_d4 = nullptr;
  uint64_t* src_off4 = nullptr;
  unsigned* err = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_main = nullptr, ev_grad = nullptr;
  // owner blocks: [2][bl][D_total] (double-buffered by step parity) + flags
  char* own = nullptr;  // cudaMalloc'd (peer path: exported over IPC)
  size_t own_bytes = 0;
  float* blocks[2] = {nullptr, nullptr};
  uint64_t* flags = nullptr;
  int parity = 0;
  uint64_t seq = 0;
  // peer path
  std::vector<char*> peer_base;  // mapped IPC bases (nullptr for self)
  float** d_peer_blocks[2] = {nullptr, nullptr};  // device arrays of N pointers
  uint64_t** d_peer_flags = nullptr;
  bool connected = false;
  // nccl path
  ncclComm_t comm = nullptr;
  ncclUniqueId uid;
  float* local_pooled = nullptr;  // [B, D_local]
  float* recv = nullptr;          // sum_s bl * D_s
  float* send = nullptr;
  std::vector<uint64_t> src_off_h;
  // gradient rows for the operator's backward: [B, D_local]
  float* grad_local = nullptr;
  uint64_t spin_limit = 1ull << 27;  // ~30 s of 200 ns polls

  ~rs_exchange() {
    if (side) cudaStreamSynchronize(side);
    if (ctx) cudaStreamSynchronize(ctx->stream);
    if (comm) rs::ex::nccl().CommDestroy(comm);
    for (char* p : peer_base)
      if (p) cudaIpcCloseMemHandle(p);
    for (void* p : {(void*)gsrc, (void*)gcol4, (void*)lmap, (void*)xcol, (void*)src_d4, (void*)src_off4,
                    (void*)err, (void*)own, (void*)d_peer_blocks[0], (void*)d_peer_blocks[1],
                    (void*)d_peer_flags, (void*)local_pooled, (void*)recv, (void*)send, (void*)grad_local})
      if (p) cudaFree(p);
    if (side) cudaStreamDestroy(side);
    if (ev_main) cudaEventDestroy(ev_main);
    if (ev_grad) cudaEventDestroy(ev_grad);
  }
};

namespace rs {

template <class T>
static T* to_device(const std::vector<T>& v, cudaStream_t st) {
  T* p = nullptr;
  RS_CUDA(cudaMalloc(&p, std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) RS_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return p;
}

static unsigned grid_for(uint64_t n) {
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(sm_count()) * 8)));
}

rs_exchange* exchange_create(rs_context* ctx, int kind, uint32_t N, uint32_t rank, uint64_t B, uint32_t J,
                             const uint32_t* dims, const uint32_t* owner) {
  if (kind != RS_EX_PEER && kind != RS_EX_NCCL) throw InvalidArgument("exchange: unknown transport");
  if (N < 1 || N > uint32_t(kMaxRanks)) throw InvalidArgument("exchange: 1 <= nranks <= 8");
  if (rank >= N) throw InvalidArgument("exchange: rank outside [0, nranks)");
  if (B == 0 || B % N) throw InvalidArgument("exchange: the global batch must be a positive multiple of nranks");
  if (J == 0 || !dims || !owner) throw InvalidArgument("exchange: no tables");
  auto* x = new rs_exchange;
  try {
    x->ctx = ctx;
    x->kind = kind;
    x->N = N;
    x->rank = rank;
    x->B = B;
    x->bl = B / N;
    x->J = J;
    x->dims.assign(dims, dims + J);
    x->owner.assign(owner, owner + J);
    x->Drank.assign(N, 0);
    for (uint32_t j = 0; j < J; ++j) {
      if (dims[j] == 0 || dims[j] % 4) throw InvalidArgument("exchange: dims must be positive multiples of 4");
      if (owner[j] >= N) throw InvalidArgument("exchange: table owner outside [0, nranks)");
      x->gcol.push_back(uint32_t(x->D_total));
      x->D_total += dims[j];
      x->Drank[owner[j]] += dims[j];
      if (owner[j] == rank) {
        x->local.push_back(j);
        x->xcol_h.push_back(x->gcol[j]);
      }
    }
    x->D_local = x->Drank[rank];
    cudaStream_t st = ctx->stream;
    // float4 column maps
    const uint32_t D4 = uint32_t(x->D_total / 4);
    std::vector<uint32_t> gsrc(D4), gcol4(D4), lmap;
    std::vector<uint32_t> within(N, 0);  // running column inside each rank's block
    for (uint32_t j = 0; j < J; ++j) {
      for (uint32_t c = 0; c < dims[j] / 4; ++c) {
        const uint32_t g = x->gcol[j] / 4 + c;
        gsrc[g] = owner[j];
        gcol4[g] = within[owner[j]] / 4 + c;
        if (owner[j] == rank) lmap.push_back(g);
      }
      within[owner[j]] += dims[j];
    }
    std::vector<uint32_t> d4(N);
    std::vector<uint64_t> off4(N + 1, 0);
    for (uint32_t r = 0; r < N; ++r) {
      d4[r] = x->Drank[r] / 4;
      off4[r + 1] = off4[r] + x->bl * d4[r];
    }
    x->src_off_h = off4;
    x->gsrc = to_device(gsrc, st);
    x->gcol4 = to_device(gcol4, st);
    x->lmap = to_device(lmap, st);
    x->xcol = to_device(x->xcol_h, st);
    x->src_d4 = to_device(d4, st);
    x->src_off4 = to_device(off4, st);
    RS_CUDA(cudaMalloc(&x->err, 4));
    RS_CUDA(cudaMemsetAsync(x->err, 0, 4, st));
    if (const char* v = getenv("RS_EXCHANGE_SPIN_LIMIT")) x->spin_limit = std::max(1ull, strtoull(v, nullptr, 10));
    RS_CUDA(cudaStreamCreateWithFlags(&x->side, cudaStreamNonBlocking));
    RS_CUDA(cudaEventCreateWithFlags(&x->ev_main, cudaEventDisableTiming));
    RS_CUDA(cudaEventCreateWithFlags(&x->ev_grad, cudaEventDisableTiming));
    // owner blocks (+ 4 KiB of flags), one allocation so one IPC handle maps it
    const size_t blk = size_t(x->bl) * x->D_total * 4;
    const size_t blk_al = (blk + 4095) / 4096 * 4096;
    x->own_bytes = 2 * blk_al + 4096;
    RS_CUDA(cudaMalloc(&x->own, x->own_bytes));
    RS_CUDA(cudaMemsetAsync(x->own, 0, x->own_bytes, st));
    x->blocks[0] = reinterpret_cast<float*>(x->own);
    x->blocks[1] = reinterpret_cast<float*>(x->own + blk_al);
    x->flags = reinterpret_cast<uint64_t*>(x->own + 2 * blk_al);
    RS_CUDA(cudaMalloc(&x->grad_local, std::max<uint64_t>(1, B * x->D_local) * 4));
    if (kind == RS_EX_NCCL) {
      RS_CUDA(cudaMalloc(&x->local_pooled, std::max<uint64_t>(1, B * x->D_local) * 4));
      RS_CUDA(cudaMalloc(&x->recv, std::max<uint64_t>(1, off4[N] * 4) * 4));
      RS_CUDA(cudaMalloc(&x->send, std::max<uint64_t>(1, off4[N] * 4) * 4));
      if (rank == 0) RS_NCCL(ex::nccl().GetUniqueId(&x->uid));
    }
    RS_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    delete x;
    throw;
  }
  return x;
}

void exchange_blob(rs_exchange* x, void* blob) {
  std::memset(blob, 0, RS_EX_BLOB_BYTES);
  if (x->kind == RS_EX_NCCL) {
    static_assert(sizeof(ncclUniqueId) <= RS_EX_BLOB_BYTES, "blob too small");
    std::memcpy(blob, &x->uid, sizeof(ncclUniqueId));
  } else {
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) <= RS_EX_BLOB_BYTES, "blob too small");
    RS_CUDA(cudaIpcGetMemHandle(&h, x->own));
    std::memcpy(blob, &h, sizeof(h));
  }
}

void exchange_connect(rs_exchange* x, const void* blobs) {
  if (x->connected) throw InvalidArgument("exchange: already connected");
  const char* b = static_cast<const char*>(blobs);
  cudaStream_t st = x->ctx->stream;
  if (x->kind == RS_EX_NCCL) {
    ncclUniqueId id;
    std::memcpy(&id, b, sizeof(id));  // rank 0's id
    RS_NCCL(ex::nccl().CommInitRank(&x->comm, int(x->N), id, int(x->rank)));
  } else {
    x->peer_base.assign(x->N, nullptr);
    std::vector<float*> pb[2];
    std::vector<uint64_t*> pf;
    const size_t blk_al = reinterpret_cast<char*>(x->blocks[1]) - reinterpret_cast<char*>(x->blocks[0]);
    for (uint32_t r = 0; r < x->N; ++r) {
      char* base = x->own;
      if (r != x->rank) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, b + size_t(r) * RS_EX_BLOB_BYTES, sizeof(h));
        void* p = nullptr;
        RS_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        base = static_cast<char*>(p);
        x->peer_base[r] = base;
      }
      pb[0].push_back(reinterpret_cast<float*>(base));
      pb[1].push_back(reinterpret_cast<float*>(base + blk_al));
      pf.push_back(reinterpret_cast<uint64_t*>(base + 2 * blk_al));
    }
    x->d_peer_blocks[0] = to_device(pb[0], st);
    x->d_peer_blocks[1] = to_device(pb[1], st);
    x->d_peer_flags = to_device(pf, st);
    RS_CUDA(cudaStreamSynchronize(st));
  }
  x->connected = true;
}

static void check_binding(rs_exchange* x, rs_emb* e) {
  if (!x->connected) throw InvalidArgument("exchange: connect it first");
  if (emb_context(e) != x->ctx) throw InvalidArgument("exchange: the operator runs on another context");
  const uint32_t T = emb_num_tables(e);
  if (T != x->local.size()) throw InvalidArgument("exchange: the operator's tables are not this rank's tables");
  for (uint32_t t = 0; t < T; ++t)
    if (emb_table_dim(e, t) != x->dims[x->local[t]])
      throw InvalidArgument("exchange: operator table dims differ from the exchange's table map");
}

static void barrier(rs_exchange* x, cudaStream_t st) {
  ++x->seq;
  ex::barrier_kernel<<<1, 32, 0, st>>>(x->d_peer_flags, x->flags, x->rank, x->N, x->seq, x->err, x->spin_limit);
  RS_COUNT(1);
  RS_LAUNCH_CHECK();
}

static unsigned take_err(rs_exchange* x) {
  unsigned h = 0;
  RS_CUDA(cudaMemcpy(&h, x->err, 4, cudaMemcpyDeviceToHost));
  if (h) RS_CUDA(cudaMemset(x->err, 0, 4));
  return h;
}

// K4 + K6 forward: this rank's tables pooled for all B samples, every row
// delivered to its sample owner.  Returns this rank's owner block.
float* exchange_forward(rs_exchange* x, rs_emb* e, const uint32_t* off, const uint32_t* idx, uint64_t* hits) {
  check_binding(x, e);
  cudaStream_t st = x->ctx->stream;
  x->parity ^= 1;
  float* mine = x->blocks[x->parity];
  if (x->kind == RS_EX_PEER) {
    if (!x->local.empty()) {
      OutMap om{};
      om.out0 = mine;  // out_row's single-destination path (N == 1)
      om.peers = x->d_peer_blocks[x->parity];
      om.xcol = x->xcol;
      om.bl = x->bl;
      om.n = x->N;
      emb_forward_map(e, x->B, off, idx, om, x->D_total, hits);
    }
    barrier(x, st);  // every owner block complete
    return mine;
  }
  // NCCL: K4 into [B, D_local] (already destination-major), send/recv, scatter
  if (!x->local.empty()) {
    OutMap om{};
    om.out0 = x->local_pooled;
    om.n = 1;
    emb_forward_map(e, x->B, off, idx, om, x->D_local, hits);
  }
  const auto& n = ex::nccl();
  RS_NCCL(n.GroupStart());
  for (uint32_t r = 0; r < x->N; ++r) {
    if (x->D_local)
      RS_NCCL(n.Send(x->local_pooled + r * x->bl * x->D_local, x->bl * x->D_local, ncclFloat32, int(r), x->comm, st));
    if (x->Drank[r])
      RS_NCCL(n.Recv(x->recv + x->src_off_h[r] * 4, x->bl * x->Drank[r], ncclFloat32, int(r), x->comm, st));
  }
  RS_NCCL(n.GroupEnd());
  const uint64_t tot = x->bl * (x->D_total / 4);
  ex::assemble_kernel<<<grid_for(tot), 256, 0, st>>>(reinterpret_cast<const float4*>(x->recv), x->src_off4,
                                                      x->src_d4, x->gsrc, x->gcol4, x->bl, uint32_t(x->D_total / 4),
                                                      reinterpret_cast<float4*>(mine));
  RS_COUNT(1);
  RS_LAUNCH_CHECK();
  return mine;
}

// K6 backward + K5: the gradients of this rank's owner block (written in
// place into the block exchange_forward returned, or copied from
// `grad_owned`) travel to the table owners on a side stream while K5 sorts.
void exchange_backward(rs_exchange* x, rs_emb* e, const uint32_t* off, const uint32_t* idx, const float* grad_owned,
                       float lr) {
  check_binding(x, e);
  cudaStream_t st = x->ctx->stream;
  float* mine = x->blocks[x->parity];
  if (grad_owned && grad_owned != mine)
    RS_CUDA(cudaMemcpyAsync(mine, grad_owned, x->bl * x->D_total * 4, cudaMemcpyDeviceToDevice, st));
  RS_CUDA(cudaEventRecord(x->ev_main, st));
  RS_CUDA(cudaStreamWaitEvent(x->side, x->ev_main, 0));
  if (x->kind == RS_EX_PEER) {
    barrier(x, x->side);  // every owner's gradients are in place
    if (!x->local.empty()) {
      const uint64_t tot = x->B * (x->D_local / 4);
      ex::pull_kernel<<<grid_for(tot), 256, 0, x->side>>>(
          reinterpret_cast<const float4* const*>(x->d_peer_blocks[x->parity]), x->lmap, x->B, x->bl,
          uint32_t(x->D_total / 4), uint32_t(x->D_local / 4), reinterpret_cast<float4*>(x->grad_local), x->err);
      RS_COUNT(1);
      RS_LAUNCH_CHECK();
    }
  } else {
    const uint64_t tot = x->bl * (x->D_total / 4);
    ex::pack_kernel<<<grid_for(tot), 256, 0, x->side>>>(reinterpret_cast<const float4*>(mine), x->src_off4,
                                                         x->src_d4, x->gsrc, x->gcol4, x->bl,
                                                         uint32_t(x->D_total / 4), reinterpret_cast<float4*>(x->send));
    RS_COUNT(1);
    RS_LAUNCH_CHECK();
    const auto& n = ex::nccl();
    RS_NCCL(n.GroupStart());
    for (uint32_t r = 0; r < x->N; ++r) {
      if (x->Drank[r])
        RS_NCCL(n.Send(x->send + x->src_off_h[r] * 4, x->bl * x->Drank[r], ncclFloat32, int(r), x->comm, x->side));
      if (x->D_local)
        RS_NCCL(n.Recv(x->grad_local + r * x->bl * x->D_local, x->bl * x->D_local, ncclFloat32, int(r), x->comm,
                       x->side));
    }
    RS_NCCL(n.GroupEnd());
  }
  RS_CUDA(cudaEventRecord(x->ev_grad, x->side));
  if (!x->local.empty()) {
    emb_set_grad_ready(e, x->ev_grad);
    emb_backward(e, x->B, off, idx, x->grad_local, lr);
  } else {
    RS_CUDA(cudaStreamWaitEvent(st, x->ev_grad, 0));
  }
  if (x->kind == RS_EX_PEER) {
    // a peer that never reached a barrier (e.g. a crashed rank): report it
    // instead of training on a partial block
    unsigned h = 0;
    RS_CUDA(cudaMemcpyAsync(&h, x->err, 4, cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    if (h) {
      take_err(x);
      throw Error(RS_ERR_INTERNAL, "exchange: a peer rank did not reach the barrier (timeout)");
    }
  }
}

// The K6 primitives on their own (rs_emb_alltoall_{fwd,bwd}): pooled rows
// [B, D_local] of this rank's tables -> its owner block [bl, D_total];
// gradients [bl, D_total] -> [B, D_local].
void alltoall_fwd(rs_exchange* x, const float* pooled_local, float* pooled_owned) {
  if (!x->connected) throw InvalidArgument("exchange: connect it first");
  cudaStream_t st = x->ctx->stream;
  if (x->kind == RS_EX_PEER) {
    x->parity ^= 1;
    const uint64_t tot = x->B * (x->D_local / 4);
    if (tot) {
      ex::push_kernel<<<grid_for(tot), 256, 0, st>>>(
          reinterpret_cast<const float4*>(pooled_local), reinterpret_cast<float4* const*>(x->d_peer_blocks[x->parity]),
          x->lmap, x->B, x->bl, uint32_t(x->D_total / 4), uint32_t(x->D_local / 4));
      RS_COUNT(1);
      RS_LAUNCH_CHECK();
    }
    barrier(x, st);
    if (pooled_owned && pooled_owned != x->blocks[x->parity])
      RS_CUDA(cudaMemcpyAsync(pooled_owned, x->blocks[x->parity], x->bl * x->D_total * 4, cudaMemcpyDeviceToDevice,
                              st));
    return;
  }
  const auto& n = ex::nccl();
  RS_NCCL(n.GroupStart());
  for (uint32_t r = 0; r < x->N; ++r) {
    if (x->D_local)
      RS_NCCL(n.Send(pooled_local + r * x->bl * x->D_local, x->bl * x->D_local, ncclFloat32, int(r), x->comm, st));
    if (x->Drank[r])
      RS_NCCL(n.Recv(x->recv + x->src_off_h[r] * 4, x->bl * x->Drank[r], ncclFloat32, int(r), x->comm, st));
  }
  RS_NCCL(n.GroupEnd());
  const uint64_t tot = x->bl * (x->D_total / 4);
  ex::assemble_kernel<<<grid_for(tot), 256, 0, st>>>(reinterpret_cast<const float4*>(x->recv), x->src_off4,
                                                      x->src_d4, x->gsrc, x->gcol4, x->bl, uint32_t(x->D_total / 4),
                                                      reinterpret_cast<float4*>(pooled_owned));
  RS_COUNT(1);
  RS_LAUNCH_CHECK();
}

void alltoall_bwd(rs_exchange* x, const float* grad_owned, float* grad_local) {
  if (!x->connected) throw InvalidArgument("exchange: connect it first");
  cudaStream_t st = x->ctx->stream;
  if (x->kind == RS_EX_PEER) {
    float* mine = x->blocks[x->parity];
    if (grad_owned && grad_owned != mine)
      RS_CUDA(cudaMemcpyAsync(mine, grad_owned, x->bl * x->D_total * 4, cudaMemcpyDeviceToDevice, st));
    barrier(x, st);
    const uint64_t tot = x->B * (x->D_local / 4);
    if (tot) {
      ex::pull_kernel<<<grid_for(tot), 256, 0, st>>>(
          reinterpret_cast<const float4* const*>(x->d_peer_blocks[x->parity]), x->lmap, x->B, x->bl,
          uint32_t(x->D_total / 4), uint32_t(x->D_local / 4), reinterpret_cast<float4*>(grad_local), x->err);
      RS_COUNT(1);
      RS_LAUNCH_CHECK();
    }
    return;
  }
  const uint64_t tot = x->bl * (x->D_total / 4);
  ex::pack_kernel<<<grid_for(tot), 256, 0, st>>>(reinterpret_cast<const float4*>(grad_owned), x->src_off4,
                                                  x->src_d4, x->gsrc, x->gcol4, x->bl, uint32_t(x->D_total / 4),
                                                  reinterpret_cast<float4*>(x->send));
  RS_COUNT(1);
  RS_LAUNCH_CHECK();
  const auto& n = ex::nccl();
  RS_NCCL(n.GroupStart());
  for (uint32_t r = 0; r < x->N; ++r) {
    if (x->Drank[r])
      RS_NCCL(n.Send(x->send + x->src_off_h[r] * 4, x->bl * x->Drank[r], ncclFloat32, int(r), x->comm, st));
    if (x->D_local)
      RS_NCCL(n.Recv(grad_local + r * x->bl * x->D_local, x->bl * x->D_local, ncclFloat32, int(r), x->comm, st));
  }
  RS_NCCL(n.GroupEnd());
}

void exchange_info(const rs_exchange* x, uint64_t* bl, uint64_t* d_total, uint64_t* d_local, float** owned) {
  if (bl) *bl = x->bl;
  if (d_total) *d_total = x->D_total;
  if (d_local) *d_local = x->D_local;
  if (owned) *owned = x->blocks[x->parity];
}

void exchange_free(rs_exchange* x) { delete x; }

}  // namespace rs
