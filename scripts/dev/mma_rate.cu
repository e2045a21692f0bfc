// Dev microbenchmark: legacy mma.sync m16n8k16 (HMMA) issue rate per SM on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int ACC>
__global__ void k(float* out, int iters) {
  float d[ACC][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c003c00u, b1 = b0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < ACC; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < ACC; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 1024 * 4 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    k<8><<<148, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    k<8><<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double mmas = 148.0 * warps * iters * 8;
    printf("warps/SM %2d: %.3f ms, %.3f mma/clk/SM @1.965GHz, %.1f TFLOPS f16\n", warps, ms,
           mmas / 148 / (ms * 1e-3 * 1.965e9), mmas * 4096 * 2 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
