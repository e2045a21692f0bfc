// Dev microbenchmark: tcgen05.mma (A from TMEM, B from smem) throughput and commit round-trip latency.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return ((uint64_t)(addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
template <int N, int MODE>   // MODE 0: TS, MODE 1: SS
__global__ void k(int blocks, int per_block, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* b = sm;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    for (int blk = 0; blk < blocks; ++blk) {
#pragma unroll 16
      for (int kk = 0; kk < per_block; ++kk) {
        const uint64_t bd = desc_sw128(su32(b) + (kk & 3) * 32);
        if (MODE == 0)
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tm + 256), "r"(tm + (kk & 15) * 8), "l"(bd), "r"(idesc), "r"(kk));
        else
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tm + 256), "l"(desc_sw128(su32(b) + 32768 + (kk & 3) * 32)), "l"(bd), "r"(idesc), "r"(kk));
      }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(&bar)) : "memory");
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar)), "r"(blk & 1) : "memory");
    }
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}
int main() {
  long long* out;
  cudaMalloc(&out, 8);
  auto run = [&](auto kern, const char* name, int blocks, int per) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    kern<<<1, 128, 64 * 1024>>>(blocks, per, out);
    kern<<<148, 128, 64 * 1024>>>(blocks, per, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("%-10s blocks %4d x %3d MMAs (commit+wait per block): %8.1f clk/block, %6.1f clk/MMA %s\n", name, blocks,
           per, (double)c / blocks, (double)c / blocks / per, e ? cudaGetErrorString(e) : "");
  };
  for (int per : {1, 16, 64, 256}) {
    run(k<16, 0>, "TS N=16", 64, per);
    run(k<16, 1>, "SS N=16", 64, per);
    run(k<128, 0>, "TS N=128", 64, per);
    run(k<128, 1>, "SS N=128", 64, per);
    run(k<256, 0>, "TS N=256", 64, per);
  }
  return 0;
}
