// Shared device helpers for the RecShard B200 hot paths (sm_100a only).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace rs {

// ---------------------------------------------------------------- errors
// Host-side exception types carrying the C-ABI status they map to
// (include/shardplan_gpu.h).  They mirror the reference's exception taxonomy
// (inc/error.hpp:38-72) so the C++ shim can rethrow the matching type.
struct Error : std::runtime_error {
  int status;
  Error(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};
struct InvalidArgument : Error {
  explicit InvalidArgument(const std::string& m) : Error(-1, m) {}
};
struct ParseError : Error {
  explicit ParseError(const std::string& m) : Error(-2, m) {}
};
struct IoError : Error {
  explicit IoError(const std::string& m) : Error(-4, m) {}
};
struct OutOfRange : Error {
  explicit OutOfRange(const std::string& m) : Error(-5, m) {}
};
struct CudaError : Error {
  explicit CudaError(const std::string& m) : Error(-8, m) {}
};

#define RS_CUDA(expr)                                                       \
  do {                                                                      \
    cudaError_t e_ = (expr);                                                \
    if (e_ != cudaSuccess)                                                  \
      throw ::rs::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_) \
                            + " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define RS_LAUNCH_CHECK() RS_CUDA(cudaGetLastError())

// Process-wide count of kernel launches issued by this library (exported as
// rs_launch_counter() so benches can report how many of OUR kernels ran).
uint64_t& launch_counter();
#define RS_COUNT(n) (::rs::launch_counter() += (n))

// ---------------------------------------------------------------- hashing
// SplitMix64 finalizer, inc/rng.hpp:27-31 (constants are the published ones).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;  // inc/rng.hpp:25

// inc/rng.hpp:61-64
__host__ __device__ __forceinline__ uint64_t derive_stream(uint64_t master,
                                                           uint64_t a,
                                                           uint64_t b) {
  uint64_t s = mix64(master ^ (kGamma * (a + 1)));
  return mix64(s ^ (0xD1B54A32D192ED03ULL * (b + 1)));
}

// First next_double() of SplitMix64(seed): inc/rng.hpp:38-44.  The u64->f64
// conversion of a 53-bit integer and the power-of-two scale are exact, so the
// device result is bit-identical to the host's.
__host__ __device__ __forceinline__ double first_double(uint64_t seed) {
  return static_cast<double>(mix64(seed + kGamma) >> 11) * 0x1.0p-53;
}

// Exact u64 % d for 1 <= d < 2^32 without a div.u64 sequence
// (inc/workload.hpp:30 computes mix64(raw) % hash_size).  m = floor((2^64-1)/d)
// is precomputed per table; q = mulhi(x, m) undershoots floor(x/d) by at most
// one, so a single conditional subtract makes the remainder exact.
struct FastMod {
  uint64_t d;
  uint64_t m;
  static FastMod make(uint64_t d) { return FastMod{d, d ? ~0ULL / d : 0}; }
};

__device__ __forceinline__ uint64_t fast_mod(uint64_t x, uint64_t d, uint64_t m) {
  uint64_t q = __umul64hi(x, m);
  uint64_t r = x - q * d;
  return r >= d ? r - d : r;
}

// ---------------------------------------------------------------- memory
__device__ __forceinline__ float4 ld_nc_f4(const float4* p) {
  float4 r;
#ifdef RS_NC_NONVOLATILE
  asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
#else
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
#endif
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint2 ld_nc_u2(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// Streaming loads: no L1 allocation, and L2 evict-first so a large input
// stream does not push resident working sets (counters, remaps) out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(r) : "l"(p), "l"(l2_evict_first_policy()));
  return r;
}
__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t* p) {
  uint64_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
               : "=l"(r) : "l"(p), "l"(l2_evict_first_policy()));
  return r;
}

// 16-byte global -> shared async copy through L2 only (LDGSTS.BYPASS).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = uint32_t(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

inline int sm_count() {
  static int n = [] {
    int dev = 0, v = kNumSMs;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace rs
