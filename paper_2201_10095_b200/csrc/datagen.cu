// Synthetic Zipf workload generator on the GPU — bench/test INPUT, not a hot
// path.  It mirrors the structure of the reference generator
// (core/src/workload.cpp:198-217: per (sample, table) SplitMix64 substream via
// derive_stream, a coverage Bernoulli, a pooling draw, k bounded-Zipf raw
// values hashed with hash_value) using the published Hormann-Derflinger
// rejection-inversion sampler.  GPU libm differs from glibc in the last ulp,
// so batches are NOT bit-identical to the reference generator's; parity
// tests therefore feed reference-generated traces, and this generator only
// produces the bench's large batches.
#include <algorithm>

#include "../../include/shardplan_gpu.h"
#include "context.cuh"

namespace rs {
namespace gen {

struct Rng {
  uint64_t s;
  __device__ uint64_t next() {
    s += kGamma;
    return mix64(s);
  }
  __device__ double next_double() { return double(next() >> 11) * 0x1.0p-53; }
  __device__ double next_open() { return (double(next() >> 12) + 0.5) * 0x1.0p-52; }
};

struct ZipfDev {
  double s, hx1, hn, thr, n;
  uint64_t card;
  uint64_t hash_size, magic;
  double mean, lambda, mu, sigma, coverage;
  int law;
  uint32_t table_id;
};

__host__ __device__ inline double helper1(double x) {
  return fabs(x) > 1e-8 ? log1p(x) / x : 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x));
}
__host__ __device__ inline double helper2(double x) {
  return fabs(x) > 1e-8 ? expm1(x) / x : 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x));
}
__host__ __device__ inline double h_int(double s, double x) {
  double lx = log(x);
  return helper2((1.0 - s) * lx) * lx;
}
__host__ __device__ inline double h_fn(double s, double x) { return exp(-s * log(x)); }
__host__ __device__ inline double h_int_inv(double s, double x) {
  double t = x * (1.0 - s);
  if (t < -1.0) t = -1.0;
  return exp(helper1(t) * x);
}

__device__ uint64_t zipf_draw(const ZipfDev& z, Rng& r) {
  if (z.card == 1) return 0;
  while (true) {
    double u = z.hn + r.next_double() * (z.hx1 - z.hn);
    double x = h_int_inv(z.s, u);
    double kd = fmin(fmax(floor(x + 0.5), 1.0), z.n);
    if (kd - x <= z.thr || u >= h_int(z.s, kd + 0.5) - h_fn(z.s, kd)) return uint64_t(kd) - 1;
  }
}

__device__ double normal_draw(Rng& r) {
  double u1 = r.next_open(), u2 = r.next_double();
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

__device__ uint32_t pooling_draw(const ZipfDev& z, Rng& r) {
  if (z.law == 0) return uint32_t(max(1.0, rint(z.mean)));
  if (z.law == 1) {  // 1 + Poisson(mean - 1)
    double lam = z.lambda;
    if (lam <= 0) return 1;
    if (lam < 30.0) {
      double L = exp(-lam), p = 1.0;
      uint32_t k = 0;
      do {
        ++k;
        p *= r.next_double();
      } while (p > L);
      return k;  // (k - 1) + 1
    }
    double x = rint(lam + sqrt(lam) * normal_draw(r));
    return uint32_t(1.0 + fmax(0.0, x));
  }
  double x = exp(z.mu + z.sigma * normal_draw(r));
  return uint32_t(fmax(1.0, rint(x)));
}

// lengths[t*B + b] (0 when the feature is absent)
__global__ void lengths_kernel(const ZipfDev* __restrict__ zs, uint32_t T, uint64_t B, uint64_t base,
                               uint64_t seed, uint32_t* __restrict__ len) {
  const uint64_t n = uint64_t(T) * B;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t t = uint32_t(i / B);
    const ZipfDev& z = zs[t];
    Rng r{derive_stream(seed, base + i % B, z.table_id)};
    uint32_t k = 0;
    if (z.coverage > 0.0 && r.next_double() < z.coverage) k = pooling_draw(z, r);
    len[i] = k;
  }
}

__global__ void fill_kernel(const ZipfDev* __restrict__ zs, uint32_t T, uint64_t B, uint64_t base,
                            uint64_t seed, const uint32_t* __restrict__ off, uint32_t* __restrict__ idx) {
  const uint64_t n = uint64_t(T) * B;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t t = uint32_t(i / B);
    const ZipfDev& z = zs[t];
    Rng r{derive_stream(seed, base + i % B, z.table_id)};
    if (!(z.coverage > 0.0 && r.next_double() < z.coverage)) continue;
    const uint32_t k = pooling_draw(z, r);
    const uint32_t o = off[i];
    for (uint32_t j = 0; j < k; ++j)
      idx[o + j] = uint32_t(fast_mod(mix64(zipf_draw(z, r)), z.hash_size, z.magic));
  }
}

struct LenIn {
  const uint32_t* p;
  __device__ __forceinline__ uint32_t operator()(size_t k) const { return p[k]; }
};
struct NzIn {
  const uint32_t* off;
  __device__ __forceinline__ uint32_t operator()(size_t k) const { return off[k + 1] != off[k]; }
};

__global__ void records_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ pos,
                               const uint32_t* __restrict__ tids, uint32_t T, uint64_t B, uint64_t base,
                               uint64_t* __restrict__ rs_, uint32_t* __restrict__ rt,
                               uint64_t* __restrict__ ro, uint32_t* __restrict__ rl) {
  const uint64_t n = uint64_t(T) * B;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t len = off[i + 1] - off[i];
    if (!len) continue;
    const uint32_t p = pos[i];
    rs_[p] = base + i % B;
    rt[p] = tids[i / B];
    ro[p] = off[i];
    rl[p] = len;
  }
}

}  // namespace gen
}  // namespace rs

namespace rs {

void gen_batch(rs_context* ctx, uint32_t T, const rs_gen_table* tabs, uint64_t B, uint64_t base,
               uint64_t seed, uint32_t* off, uint32_t* idx, uint64_t cap, uint64_t* total) {
  using namespace gen;
  if (T == 0 || B == 0) throw InvalidArgument("gen_batch: empty batch");
  cudaStream_t st = ctx->stream;
  std::vector<ZipfDev> zs(T);
  for (uint32_t t = 0; t < T; ++t) {
    const rs_gen_table& g = tabs[t];
    if (g.hash_size == 0 || g.cardinality == 0) throw InvalidArgument("gen_batch: empty table");
    ZipfDev& z = zs[t];
    z.s = g.zipf_exponent;
    z.card = g.cardinality;
    z.n = double(g.cardinality);
    z.hx1 = h_int(z.s, 1.5) - 1.0;
    z.hn = h_int(z.s, z.n + 0.5);
    z.thr = 2.0 - h_int_inv(z.s, h_int(z.s, 2.5) - h_fn(z.s, 2.0));
    z.hash_size = g.hash_size;
    z.magic = FastMod::make(g.hash_size).m;
    z.mean = g.mean_pooling < 1.0 ? 1.0 : g.mean_pooling;
    z.lambda = z.mean - 1.0;
    z.sigma = 0.75;
    z.mu = std::log(z.mean) - 0.5 * z.sigma * z.sigma;
    z.coverage = g.coverage;
    z.law = g.pooling_law;
    z.table_id = g.table_id;
  }
  const uint64_t n = uint64_t(T) * B;
  Scratch scr = ctx->scratch(sizeof(ZipfDev) * T + n * 4 + scan_scratch_bytes(n, 4) + (4 << 20));
  ZipfDev* d_z = stage(zs.data(), T, false, scr, st);
  uint32_t* len = scr.take<uint32_t>(n);
  const unsigned g = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(sm_count()) * 16));
  lengths_kernel<<<g, 256, 0, st>>>(d_z, T, B, base, seed, len);
  exclusive_scan<uint32_t>(LenIn{len}, n, off, off + n, scr, st);
  uint32_t h_total = 0;
  RS_CUDA(cudaMemcpyAsync(&h_total, off + n, 4, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  *total = h_total;
  if (h_total > cap) throw InvalidArgument("gen_batch: capacity too small for the batch");
  fill_kernel<<<g, 128, 0, st>>>(d_z, T, B, base, seed, off, idx);
  RS_LAUNCH_CHECK();
}

void kjt_to_records(rs_context* ctx, uint32_t T, const uint32_t* tids, uint64_t B, uint64_t base,
                    const uint32_t* off, uint64_t* rs_, uint32_t* rt, uint64_t* ro, uint32_t* rl,
                    uint64_t* R) {
  using namespace gen;
  cudaStream_t st = ctx->stream;
  const uint64_t n = uint64_t(T) * B;
  Scratch scr = ctx->scratch(n * 4 + T * 4 + scan_scratch_bytes(n, 4) + (4 << 20));
  uint32_t* pos = scr.take<uint32_t>(n + 1);
  uint32_t* d_t = stage(tids, T, false, scr, st);
  exclusive_scan<uint32_t>(NzIn{off}, n, pos, pos + n, scr, st);
  const unsigned g = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(sm_count()) * 16));
  records_kernel<<<g, 256, 0, st>>>(off, pos, d_t, T, B, base, rs_, rt, ro, rl);
  RS_LAUNCH_CHECK();
  uint32_t h = 0;
  RS_CUDA(cudaMemcpyAsync(&h, pos + n, 4, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  *R = h;
}

}  // namespace rs

namespace rs {
void set_error(const std::string& m);
}

extern "C" int rs_gen_batch(rs_context* ctx, uint32_t T, const rs_gen_table* tabs, uint64_t B,
                            uint64_t base, uint64_t seed, uint32_t* off, uint32_t* idx, uint64_t cap,
                            uint64_t* total) {
  try {
    rs::gen_batch(ctx, T, tabs, B, base, seed, off, idx, cap, total);
    return RS_OK;
  } catch (const rs::Error& e) {
    rs::set_error(e.what());
    return e.status;
  } catch (const std::exception& e) {
    rs::set_error(e.what());
    return RS_ERR_INTERNAL;
  }
}

extern "C" int rs_kjt_to_records(rs_context* ctx, uint32_t T, const uint32_t* tids, uint64_t B,
                                 uint64_t base, const uint32_t* off, uint64_t* rs_, uint32_t* rt,
                                 uint64_t* ro, uint32_t* rl, uint64_t* R) {
  try {
    rs::kjt_to_records(ctx, T, tids, B, base, off, rs_, rt, ro, rl, R);
    return RS_OK;
  } catch (const rs::Error& e) {
    rs::set_error(e.what());
    return e.status;
  } catch (const std::exception& e) {
    rs::set_error(e.what());
    return RS_ERR_INTERNAL;
  }
}
