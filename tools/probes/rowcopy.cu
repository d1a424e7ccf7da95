// Random-row read+write ceiling on B200: out[i] = in[perm[i]] (gather) and
// W[perm[i]] += 1 (RMW) for 256/512 B rows, warp-per-row with U rows in
// flight per warp.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a rowcopy.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int G, int U>
__global__ void __launch_bounds__(256) gather(const float4* __restrict__ in, const unsigned* __restrict__ perm,
                                              float4* __restrict__ out, unsigned n, unsigned V) {
  const int lane = threadIdx.x & 31, grp = lane / G, lg = lane % G;
  const unsigned BPW = 32 / G;
  const unsigned nw = gridDim.x * blockDim.x / 32;
  for (unsigned r0 = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * BPW * U; r0 < n; r0 += nw * BPW * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned r = r0 + u * BPW + grp;
      v[u] = r < n ? __ldg(in + size_t(perm[r]) * V + lg) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned r = r0 + u * BPW + grp;
      if (r < n) out[size_t(r) * V + lg] = v[u];
    }
  }
}
template <int G, int U>
__global__ void __launch_bounds__(256) rmw(float4* __restrict__ W, const unsigned* __restrict__ perm, unsigned n,
                                           unsigned V) {
  const int lane = threadIdx.x & 31, grp = lane / G, lg = lane % G;
  const unsigned BPW = 32 / G;
  const unsigned nw = gridDim.x * blockDim.x / 32;
  for (unsigned r0 = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * BPW * U; r0 < n; r0 += nw * BPW * U) {
    float4 v[U];
    size_t a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned r = r0 + u * BPW + grp;
      a[u] = r < n ? size_t(perm[r]) * V + lg : 0;
      v[u] = r < n ? W[a[u]] : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned r = r0 + u * BPW + grp;
      if (r < n) W[a[u]] = make_float4(v[u].x + 1, v[u].y + 1, v[u].z + 1, v[u].w + 1);
    }
  }
}

template <int G, int U>
void run(float4* W, unsigned rows, unsigned* perm, unsigned n, float4* out, int sms) {
  const unsigned V = G;  // dim/4 = G lanes
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  for (int occ : {4, 8}) {
    unsigned grid = sms * occ;
    gather<G, U><<<grid, 256>>>(W, perm, out, n, V);
    cudaEventRecord(s);
    for (int i = 0; i < 10; ++i) gather<G, U><<<grid, 256>>>(W, perm, out, n, V);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    ms /= 10;
    double by = double(n) * V * 16 * 2;
    printf("gather rowB=%u U=%d occ=%d: %.3f ms %.0f GB/s (rd+wr)\n", V * 16, U, occ, ms, by / ms / 1e6);
    rmw<G, U><<<grid, 256>>>(W, perm, n, V);
    cudaEventRecord(s);
    for (int i = 0; i < 10; ++i) rmw<G, U><<<grid, 256>>>(W, perm, n, V);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    ms /= 10;
    printf("rmw    rowB=%u U=%d occ=%d: %.3f ms %.0f GB/s (rd+wr)\n", V * 16, U, occ, ms, by / ms / 1e6);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned rows = 16u << 20, n = 4u << 20;
  float4* W;
  float4* out;
  unsigned* perm;
  cudaMalloc(&W, size_t(rows) * 32 * 16);
  cudaMalloc(&out, size_t(n) * 32 * 16);
  cudaMalloc(&perm, n * 4);
  std::vector<unsigned> p(rows);
  for (unsigned i = 0; i < rows; ++i) p[i] = i;
  std::shuffle(p.begin(), p.end(), std::mt19937(1));
  cudaMemcpy(perm, p.data(), n * 4, cudaMemcpyHostToDevice);
  run<32, 2>(W, rows, perm, n, out, sms);
  run<32, 4>(W, rows, perm, n, out, sms);
  run<32, 8>(W, rows, perm, n, out, sms);
  run<16, 4>(W, rows, perm, n, out, sms);
  run<16, 8>(W, rows, perm, n, out, sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
