// Dev microbenchmark: how to stream HBM into SMs fastest on B200.
//  mode 0: one thread per CTA keeps R bulk copies (cp.async.bulk, S bytes each) in flight (pure TMA)
//  mode 1: like mode 0 but all warps wait on each slot + release counter; last releaser refills (GEMV ring)
//  mode 2: LDG.128 grid-stride, U loads in flight per thread
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mexp(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
template <int MODE>
__global__ void k(const uint8_t* __restrict__ buf, size_t per_cta, int S, int R, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)sm;
  int* rel = (int*)(sm + 256);
  uint8_t* ring = sm + 1024;
  const uint8_t* src = buf + blockIdx.x * per_cta;
  const int nch = (int)(per_cta / S);
  uint32_t acc = 0;
  if (MODE == 2) {
    const uint4* p = (const uint4*)src;
    const size_t n = per_cta / 16;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x * 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (i + u * blockDim.x < n) ? __ldcs(p + i + u * blockDim.x) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678) out[0] = acc;
    return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < R; ++s) { minit(&full[s], 1); rel[s] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;");
    for (int s = 0; s < R && s < nch; ++s) { mexp(&full[s], S); bulk(ring + s * S, src + (size_t)s * S, S, &full[s]); }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (MODE == 0) {
    if (threadIdx.x == 0) {
      for (int c = 0; c < nch; ++c) {
        const int s = c % R;
        mwait(&full[s], (c / R) & 1);
        acc ^= *(const uint32_t*)(ring + s * S);
        if (c + R < nch) { mexp(&full[s], S); bulk(ring + s * S, src + (size_t)(c + R) * S, S, &full[s]); }
      }
    }
  } else {
    for (int c = 0; c < nch; ++c) {
      const int s = c % R;
      mwait(&full[s], (c / R) & 1);
      acc ^= *(const uint32_t*)(ring + s * S + (warp * 32 + lane) * 16 % S);
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&rel[s], 1) == nw - 1) {
          rel[s] = 0;
          if (c + R < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mexp(&full[s], S); bulk(ring + s * S, src + (size_t)(c + R) * S, S, &full[s]);
          }
        }
      }
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}
int main() {
  size_t total = (size_t)1 << 30;
  uint8_t* buf; uint32_t* out;
  cudaMalloc(&buf, total); cudaMemset(buf, 1, total); cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](int mode, int grid, int threads, int S, int R) {
    size_t per = (total / grid) / 16896 * 16896;
    if (mode != 2) per = per / S * S;
    size_t smem = 1024 + (size_t)S * R;
    void (*f)(const uint8_t*, size_t, int, int, uint32_t*) = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (mode == 2) smem = 0;
    f<<<grid, threads, smem>>>(buf, per, S, R, out);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) f<<<grid, threads, smem>>>(buf, per, S, R, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("mode %d grid %4d thr %3d S %6d R %2d inflight/CTA %7zu: %7.1f GB/s %s\n", mode, grid, threads, S, R,
           (size_t)S * R, 5.0 * per * grid / (ms * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
  };
  auto small = [&](int mode, int threads, int S, int R, size_t per) {
    void (*f)(const uint8_t*, size_t, int, int, uint32_t*) = mode == 0 ? k<0> : k<1>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    size_t smem = 1024 + (size_t)S * R;
    const int reps = 50;
    for (int i = 0; i < 3; ++i) f<<<148, threads, smem>>>(buf + (i % 8) * 148 * per, per, S, R, out);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) f<<<148, threads, smem>>>(buf + (i % 8) * 148 * per, per, S, R, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("short launches: mode %d thr %d S %d R %d per-CTA %zu KB (%.1f MB/launch): %.2f us/launch = %.1f GB/s\n", mode,
           threads, S, R, per / 1024, per * 148 / 1e6, ms * 1e3 / reps, (double)per * 148 * reps / (ms * 1e-3) / 1e9);
  };
  for (size_t per : {29568UL, 78144UL, 118272UL, 409728UL}) {
    small(0, 128, 16896, 6, per / 16896 * 16896);
    small(1, 512, 16896, 6, per / 16896 * 16896);
  }
  if (getenv("SHORT_ONLY")) return 0;
  for (int grid : {148, 296})
    for (int S : {4224, 8448, 16896})
      for (int R : {2, 4, 6, 8, 12})
        if ((size_t)S * R + 1024 <= 227 * 1024 / (grid / 148)) run(0, grid, 128, S, R);
  for (int S : {8448, 16896}) for (int R : {4, 6, 8, 12}) if ((size_t)S * R <= 220000) run(1, 148, 512, S, R);
  for (int grid : {148, 296, 592, 1184}) for (int thr : {256, 512, 1024}) run(2, grid, thr, 0, 0);
  return 0;
}
