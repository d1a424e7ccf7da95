// Zero-copy (mapped pinned host memory) gather bandwidth vs host-buffer size,
// access pattern and warps in flight.  Diagnostic only.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void gather(const float4* __restrict__ host, const uint32_t* __restrict__ rows, uint64_t n,
                       float4* __restrict__ out, int V) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 4; i < n; i += nw * 4) {
    float4 x[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (i + r < n && lane < V) x[r] = host[uint64_t(rows[i + r]) * V + lane];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (i + r < n && lane < V) out[(i + r) * V + lane] = x[r];
  }
}

int main(int argc, char** argv) {
  const int V = 32;  // 512 B rows
  std::vector<double> sizes_gb = {1, 16, 48};
  const uint64_t n = 1 << 17;  // rows per launch (64 MB)
  float4* out;
  cudaMalloc(&out, n * V * 16);
  uint32_t* d_rows;
  cudaMalloc(&d_rows, n * 4);
  for (double gb : sizes_gb) {
    const uint64_t bytes = uint64_t(gb * (1ull << 30));
    const uint64_t nrows = bytes / (V * 16);
    void* h;
    if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
      printf("alloc %.0f GB failed\n", gb);
      continue;
    }
    // touch so pages exist
    for (uint64_t o = 0; o < bytes; o += 4096) ((char*)h)[o] = 1;
    float4* dh;
    cudaHostGetDevicePointer((void**)&dh, h, 0);
    std::vector<uint32_t> rows(n);
    for (int pat = 0; pat < 2; ++pat) {
      uint64_t s = 12345;
      for (uint64_t i = 0; i < n; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        rows[i] = pat == 0 ? uint32_t((s >> 33) % nrows) : uint32_t(i % nrows);
      }
      cudaMemcpy(d_rows, rows.data(), n * 4, cudaMemcpyHostToDevice);
      for (int blocks : {148, 148 * 4, 148 * 8}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        gather<<<blocks, 256>>>(dh, d_rows, n, out, V);
        cudaEventRecord(a);
        for (int k = 0; k < 3; ++k) gather<<<blocks, 256>>>(dh, d_rows, n, out, V);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("host %5.0f GB  %s  blocks %4d: %.1f GB/s\n", gb, pat ? "seq   " : "random", blocks,
               3.0 * n * V * 16 / (ms / 1e3) / 1e9);
      }
    }
    cudaFreeHost(h);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
