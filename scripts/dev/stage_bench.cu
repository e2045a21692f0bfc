// Dev microbenchmark: latency of one s8_stage_block call (one warp, one 256-column block).
#include "../../paper_2506_23025_b200/csrc/gemv_s8.cu"
#include <cstdio>
namespace tr {
void set_error(const char*, ...) {}
int sm_count() { return 148; }
}
__global__ void kst(float* out, long long* cyc, int reps) {
  __shared__ __align__(128) uint8_t xs[4096];
  __shared__ int32_t ncs[64];
  __shared__ float fsc[16];
  const int lane = threadIdx.x & 31;
  float f[8];
  for (int e = 0; e < 8; ++e) f[e] = out[lane * 8 + e];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    tr::s8_stage_block(f, xs, ncs, fsc, 1, r & 3, 0);
    f[0] += fsc[r & 3];   // serialize calls
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  if (f[0] == 1234.5f) out[0] = ncs[0];
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 8 * 148);
  cudaMemset(out, 0, 4096 * 4);
  for (int w : {1, 4, 16}) {
    kst<<<1, 32 * w>>>(out, cyc, 100);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("warps %2d: %lld cycles per s8_stage_block (err %s)\n", w, c, cudaGetErrorString(cudaGetLastError()));
  }
}
