// Dev microbenchmark: tcgen05.st (registers -> TMEM) bandwidth per SM, 32x32b.x32 shape, as K5's
// decode warps use it (each warp writes its 32-lane quadrant, 32 columns x 4 B per lane per store).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int iters, long long* out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 33 + i;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col0 = (warp >> 2) * 64;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n"
          ::"r"(tm + lane_off + ((col0 + c * 32 + (it & 1) * 128) & 511)), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
            "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
            "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
            "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
          : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    r[it & 31] += it;
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}
int main() {
  long long* out;
  cudaMalloc(&out, 8 * 148);
  const int iters = 4096;
  for (int warps : {4, 8}) {
    k<<<148, warps * 32>>>(iters, out);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)warps * 32 * 32 * 4 * 2 * iters;   // per SM
    printf("warps %d: %.1f B/clk/SM TMEM store (one 64 KB 128x256 fp16 A block: %.0f clk)  err=%s\n", warps,
           bytes / c, 65536.0 / (bytes / c), cudaGetErrorString(cudaGetLastError()));
  }
}
