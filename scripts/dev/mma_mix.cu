// Dev microbenchmark: mma.sync m16n8k16 throughput when interleaved with LOP3 decode work
// (the GEMV inner loop's mix: per "unit" 16 HMMA into 4 accumulators + ALU ops).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int ALU>
__global__ void k(float* out, int iters, uint32_t seed) {
  float d[4][4] = {};
  uint32_t w0 = threadIdx.x * seed, w1 = w0 * 3, w2 = w0 * 5, w3 = w0 * 7, b0 = 0x3c003c00u, b1 = b0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t a[4];
        const uint32_t m = 0x00030003u << (2 * j);
        if (ALU) {
          a[0] = (w0 >> s) & m; a[1] = (w1 >> s) & m; a[2] = (w2 >> s) & m; a[3] = (w3 >> s) & m;
#pragma unroll
          for (int x = 0; x < ALU - 1; ++x) { w0 ^= w1 + x; w1 ^= w2; }
        } else {
          a[0] = w0; a[1] = w1; a[2] = w2; a[3] = w3;
        }
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
      }
    }
    w2 += i; w3 ^= i;
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 1024 * 4 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 2048;
  auto run = [&](auto kern, int alu, int warps) {
    kern<<<148, warps * 32>>>(out, 8, 3);
    cudaEventRecord(e0);
    kern<<<148, warps * 32>>>(out, iters, 3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double mmas = 148.0 * warps * iters * 16;
    printf("ALU/mma %d warps/SM %2d: %.3f mma/clk/SM, %.2f instr/clk/SM (approx)\n", alu, warps,
           mmas / 148 / (ms * 1e-3 * 1.965e9), mmas * (1 + (alu ? 4 + 2 * (alu - 1) : 0)) / 148 / (ms * 1e-3 * 1.965e9));
  };
  for (int w : {8, 16, 32}) {
    run(k<0>, 0, w);
    run(k<1>, 1, w);
    run(k<3>, 3, w);
  }
  return 0;
}
