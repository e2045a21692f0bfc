// Dev microbenchmark (not part of the product): achievable HBM read bandwidth
// for the GEMV's access patterns with a register ring of S 128-bit loads.
//   pattern 0: T16 tile-major stream -- warp w owns tile w, block b at (b*n_tiles + w) KB
//   pattern 1: contiguous stream     -- warp w owns a contiguous range of KB chunks
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int S>
__global__ void k_stream(const uint4* __restrict__ w, int n_tiles, int nb, int pattern, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const int tile = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (tile >= n_tiles) return;
  uint4 r[S], r2[S];
  uint32_t acc = 0;
  auto addr = [&](int b) -> const uint4* {
    if (pattern == 0) return w + ((int64_t)b * n_tiles + tile) * 64 + lane;
    return w + ((int64_t)tile * nb + b) * 64 + lane;
  };
#pragma unroll
  for (int s = 0; s < S; ++s) if (s < nb) { r[s] = ldg(addr(s)); r2[s] = ldg(addr(s) + 32); }
  for (int base = 0; base < nb; base += S) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      int b = base + s;
      if (b < nb) {
        acc ^= r[s].x ^ r[s].y ^ r[s].z ^ r[s].w;
        acc += r2[s].x ^ r2[s].w;
        if (b + S < nb) { r[s] = ldg(addr(b + S)); r2[s] = ldg(addr(b + S) + 32); }
      }
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int S>
float run(const uint4* w, int n_tiles, int nb, int pattern, int warps, uint32_t* out) {
  int threads = warps * 32;
  int grid = (n_tiles + warps - 1) / warps;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k_stream<S><<<grid, threads>>>(w, n_tiles, nb, pattern, out);
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) k_stream<S><<<grid, threads>>>(w, n_tiles, nb, pattern, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  // 28672 x 8192 TQ2: n_tiles = 1792, nb = 32 -> 58.7 MB; use 4 copies to defeat L2 by rotating? use one big buffer
  const int n_tiles = 1792 * 4, nb = 32;   // 235 MB > L2
  size_t bytes = (size_t)n_tiles * nb * 1024;
  uint4* w;
  uint32_t* out;
  cudaMalloc(&w, bytes);
  cudaMalloc(&out, 16);
  cudaMemset(w, 1, bytes);
  for (int pattern = 0; pattern < 2; ++pattern)
    for (int warps : {4, 8}) {
      float t2 = run<2>(w, n_tiles, nb, pattern, warps, out);
      float t4 = run<4>(w, n_tiles, nb, pattern, warps, out);
      float t8 = run<8>(w, n_tiles, nb, pattern, warps, out);
      printf("pattern %d warps/cta %d: S=2 %.0f GB/s  S=4 %.0f GB/s  S=8 %.0f GB/s\n", pattern, warps,
             bytes / t2 / 1e6, bytes / t4 / 1e6, bytes / t8 / 1e6);
    }
  return 0;
}
