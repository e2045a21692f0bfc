// Dev microbenchmark #2: which async-copy mechanism streams HBM fastest into a
// per-warp shared-memory ring (GEMV weight feed)?  Each warp owns a contiguous
// range of 1 KB units and consumes them in order (XOR-reduce + optional dummy ALU work).
//   mode 0: TMA bulk copy, 1 unit (1 KB) per op
//   mode 1: TMA bulk copy, 4 units (4 KB) per op
//   mode 2: cp.async 16 B per lane (LDGSTS), commit/wait groups
//   mode 3: LDG.128 into a register ring
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(d)), "l"(s), "r"(n), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ uint4 ldg(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int MODE, int NS, int WORK>
__global__ void k(const uint8_t* __restrict__ w, int units_per_warp, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp;
  const uint8_t* base = w + (size_t)gw * units_per_warp * 1024;
  uint64_t* bars = (uint64_t*)sm + warp * NS;
  uint8_t* ring = sm + 4096 + warp * NS * 4096;
  uint32_t acc = 0;
  const int U = units_per_warp;
  if (MODE == 0 || MODE == 1) {
    const int per = MODE == 0 ? 1 : 4;          // units per op
    const int ops = U / per;
    if (lane == 0) {
      for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      for (int s = 0; s < NS && s < ops; ++s) {
        mbar_expect_tx(&bars[s], per * 1024);
        bulk(ring + s * 4096, base + (size_t)s * per * 1024, per * 1024, &bars[s]);
      }
    }
    __syncwarp();
    for (int i = 0; i < ops; ++i) {
      const int s = i % NS;
      mbar_wait(&bars[s], (i / NS) & 1);
      for (int q = 0; q < per; ++q) {
        uint4 a = *(const uint4*)(ring + s * 4096 + q * 1024 + lane * 16);
        uint4 b = *(const uint4*)(ring + s * 4096 + q * 1024 + 512 + lane * 16);
        acc ^= a.x ^ b.y;
#pragma unroll
        for (int r = 0; r < WORK; ++r) acc = acc * 3 + (a.y >> r);
      }
      __syncwarp();
      if (lane == 0 && i + NS < ops) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(&bars[s], per * 1024);
        bulk(ring + s * 4096, base + (size_t)(i + NS) * per * 1024, per * 1024, &bars[s]);
      }
    }
  } else if (MODE == 2) {
    // cp.async 16 B per lane, 2 per unit; NS units in flight (1 KB slots)
    for (int s = 0; s < NS && s < U; ++s) {
      const uint8_t* src = base + (size_t)s * 1024;
      uint8_t* dst = ring + s * 1024;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + lane * 16)), "l"(src + lane * 16));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + 512 + lane * 16)), "l"(src + 512 + lane * 16));
      asm volatile("cp.async.commit_group;\n");
    }
    for (int i = 0; i < U; ++i) {
      const int s = i % NS;
      asm volatile("cp.async.wait_group %0;\n" ::"n"(NS - 1));
      __syncwarp();
      uint4 a = *(const uint4*)(ring + s * 1024 + lane * 16);
      uint4 b = *(const uint4*)(ring + s * 1024 + 512 + lane * 16);
      acc ^= a.x ^ b.y;
#pragma unroll
      for (int r = 0; r < WORK; ++r) acc = acc * 3 + (a.y >> r);
      __syncwarp();
      if (i + NS < U) {
        const uint8_t* src = base + (size_t)(i + NS) * 1024;
        uint8_t* dst = ring + s * 1024;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + lane * 16)), "l"(src + lane * 16));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + 512 + lane * 16)), "l"(src + 512 + lane * 16));
      }
      asm volatile("cp.async.commit_group;\n");
    }
  } else {
    uint4 ra[NS], rb[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s < U) { ra[s] = ldg(base + (size_t)s * 1024 + lane * 16); rb[s] = ldg(base + (size_t)s * 1024 + 512 + lane * 16); }
    for (int i0 = 0; i0 < U; i0 += NS) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int i = i0 + s;
        if (i < U) {
          acc ^= ra[s].x ^ rb[s].y;
#pragma unroll
          for (int r = 0; r < WORK; ++r) acc = acc * 3 + (ra[s].y >> r);
          if (i + NS < U) { ra[s] = ldg(base + (size_t)(i + NS) * 1024 + lane * 16); rb[s] = ldg(base + (size_t)(i + NS) * 1024 + 512 + lane * 16); }
        }
      }
    }
  }
  if (acc == 0x9e3779b9u) out[0] = acc;
}

template <int MODE, int NS, int WORK>
void run(const uint8_t* w, size_t bytes, int warps_per_cta, int ctas_per_sm, uint32_t* out, const char* name) {
  const int ctas = 148 * ctas_per_sm;
  const int total_warps = ctas * warps_per_cta;
  const int upw = (int)(bytes / 1024 / total_warps) / 4 * 4;
  const size_t smem = 4096 + (size_t)warps_per_cta * NS * 4096;
  auto kern = k<MODE, NS, WORK>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) kern<<<ctas, warps_per_cta * 32, smem>>>(w, upw, out);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) kern<<<ctas, warps_per_cta * 32, smem>>>(w, upw, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  double moved = (double)upw * 1024 * total_warps;
  printf("%-34s warps/cta %2d ctas/sm %d NS %d work %3d: %7.0f GB/s  %s\n", name, warps_per_cta, ctas_per_sm, NS, WORK,
         moved / (ms / 10) / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  size_t bytes = (size_t)1 << 30;
  uint8_t* w;
  uint32_t* out;
  cudaMalloc(&w, bytes);
  cudaMalloc(&out, 16);
  cudaMemset(w, 3, bytes);
  run<0, 8, 0>(w, bytes, 8, 2, out, "tma 1KB/op");
  run<0, 4, 0>(w, bytes, 8, 2, out, "tma 1KB/op");
  run<1, 4, 0>(w, bytes, 8, 2, out, "tma 4KB/op");
  run<1, 2, 0>(w, bytes, 8, 2, out, "tma 4KB/op");
  run<1, 4, 0>(w, bytes, 4, 2, out, "tma 4KB/op");
  run<2, 8, 0>(w, bytes, 8, 2, out, "cp.async 16B");
  run<2, 16, 0>(w, bytes, 8, 1, out, "cp.async 16B");
  run<3, 4, 0>(w, bytes, 8, 2, out, "ldg ring");
  run<3, 8, 0>(w, bytes, 8, 2, out, "ldg ring");
  run<3, 4, 0>(w, bytes, 4, 4, out, "ldg ring");
  // with ~150 dependent ALU ops per KB (GEMV-like work)
  run<1, 4, 150>(w, bytes, 8, 2, out, "tma 4KB/op +work");
  run<2, 8, 150>(w, bytes, 8, 2, out, "cp.async 16B +work");
  run<3, 4, 150>(w, bytes, 8, 2, out, "ldg ring +work");
  run<3, 4, 150>(w, bytes, 4, 4, out, "ldg ring +work");
  return 0;
}
