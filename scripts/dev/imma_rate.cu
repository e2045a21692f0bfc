// Dev microbenchmark: legacy mma.sync m16n8k32 u8.s8 -> s32 (IMMA) issue rate per SM on B200,
// alone and interleaved with 4 LOP3 per MMA (the int8-slice GEMV inner loop's mix).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int ACC, int ALU>
__global__ void k(int* out, int iters, uint32_t seed) {
  int d[ACC][4] = {};
  uint32_t w0 = threadIdx.x * seed, w1 = w0 * 3, w2 = w0 * 5, w3 = w0 * 7, b0 = 0x01020304u * seed, b1 = b0 ^ 0x55;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < ACC; ++j) {
      uint32_t a[4];
      if (ALU) {
        const uint32_t m = 0x03030303u << (2 * (j & 3));
        a[0] = w0 & m; a[1] = w1 & m; a[2] = w2 & m; a[3] = w3 & m;
      } else {
        a[0] = w0; a[1] = w1; a[2] = w2; a[3] = w3;
      }
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(d[j][0]), "+r"(d[j][1]), "+r"(d[j][2]), "+r"(d[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    if (ALU) { w0 += i; w1 ^= i; w2 += w0; w3 ^= w1; }
  }
  int s = 0;
#pragma unroll
  for (int j = 0; j < ACC; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ACC>
__global__ void kh(float* out, int iters) {
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
  int* out;
  cudaMalloc(&out, 148 * 1024 * 4 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048;
  auto timeit = [&](auto launch, double mmas, const char* name, int warps) {
    launch(8);
    cudaEventRecord(e0);
    launch(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-22s warps/SM %2d: %.3f mma/clk/SM  (%.3f ms)  err=%s\n", name, warps, mmas / 148 / (ms * 1e-3 * 1.965e9), ms,
           cudaGetErrorString(cudaGetLastError()));
  };
  // dependent-chain latency: ACC independent accumulators per warp, one warp per SMSP
  timeit([&](int it) { k<1, 0><<<148, 128>>>(out, it, 3); }, 148.0 * 4 * iters * 1, "imma chain x1", 4);
  timeit([&](int it) { k<2, 0><<<148, 128>>>(out, it, 3); }, 148.0 * 4 * iters * 2, "imma chain x2", 4);
  timeit([&](int it) { k<4, 0><<<148, 128>>>(out, it, 3); }, 148.0 * 4 * iters * 4, "imma chain x4", 4);
  timeit([&](int it) { kh<1><<<148, 128>>>((float*)out, it); }, 148.0 * 4 * iters * 1, "hmma chain x1", 4);
  timeit([&](int it) { kh<4><<<148, 128>>>((float*)out, it); }, 148.0 * 4 * iters * 4, "hmma chain x4", 4);
  timeit([&](int it) { k<1, 0><<<148, 512>>>(out, it, 3); }, 148.0 * 16 * iters * 1, "imma chain x1", 16);
  timeit([&](int it) { k<2, 0><<<148, 512>>>(out, it, 3); }, 148.0 * 16 * iters * 2, "imma chain x2", 16);
  for (int w : {4, 8, 16, 32}) {
    timeit([&](int it) { k<8, 0><<<148, w * 32>>>(out, it, 3); }, 148.0 * w * iters * 8, "imma k32 u8s8", w);
    timeit([&](int it) { k<8, 1><<<148, w * 32>>>(out, it, 3); }, 148.0 * w * iters * 8, "imma k32 +4 LOP3", w);
    timeit([&](int it) { kh<8><<<148, w * 32>>>((float*)out, it); }, 148.0 * w * iters * 8, "hmma k16 f16", w);
  }
  return 0;
}
