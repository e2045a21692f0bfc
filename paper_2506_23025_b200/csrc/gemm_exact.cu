// Parity mode (K9): the reference matmul reproduced bit-for-bit on the GPU.
//
// Reference: _kernels.pyx:136-227 (_accumulate_row, gemm_tq2, gemm_tq1) with
// the arithmetic contract of _kernels_py.py:17-26: per block the terms
// +x / -x / +0.0 are collapsed by the fixed adjacent-pair tree
// t[i] <- t[2i] + t[2i+1] (8 levels), then acc = acc + s * T in float32,
// blocks ascending, acc starting at +0.0, no FMA.  A warp owns one
// (row, activation vector) pair; lane l holds block elements 8l..8l+7, so
// tree levels 1-3 run inside the lane and levels 4-8 are xor-shuffles -- the
// same pairings as the reference tree (fp add is commutative, so both lanes
// of a pair hold the identical node value).
#include "common.cuh"

namespace tr {

__device__ __forceinline__ float term(uint32_t d, float x) {
  return d == 2 ? x : (d == 0 ? -x : 0.0f);
}

template <int FMT>
__global__ void k_gemm_exact(const uint8_t* __restrict__ payload, const float* __restrict__ scales,
                             const float* __restrict__ x, float* __restrict__ out, int64_t rows, int64_t nb,
                             int64_t batch, int64_t row0, int64_t row1) {
  __shared__ uint8_t sdig[8][264];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nrows = row1 - row0;
  int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (; item < nrows * batch; item += nwarps) {
    const int64_t r = row0 + item % nrows, j = item / nrows;
    const float* xj = x + j * nb * kBlock;
    float acc = 0.0f;
    for (int64_t b = 0; b < nb; ++b) {
      uint32_t dg[8];
      if (FMT == kFmtTq2) {
        uint32_t w = *reinterpret_cast<const uint16_t*>(payload + (r * nb + b) * kTq2Payload + 2 * lane);
#pragma unroll
        for (int k = 0; k < 8; ++k) dg[k] = (w >> (2 * k)) & 3u;
      } else {
        const uint8_t* p = payload + (r * nb + b) * kTq1Payload;
        for (int cidx = lane; cidx < kTq1Payload; cidx += 32) {
          uint32_t s = p[cidx];
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            uint32_t prod = s * 3u;
            sdig[wib][5 * cidx + q] = (uint8_t)(prod >> 8);
            s = prod & 0xFFu;
          }
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) dg[k] = sdig[wib][8 * lane + k];
        __syncwarp();
      }
      const float4* xs = reinterpret_cast<const float4*>(xj + b * kBlock + 8 * lane);
      float4 xa = xs[0], xb = xs[1];
      float t0 = __fadd_rn(term(dg[0], xa.x), term(dg[1], xa.y));
      float t1 = __fadd_rn(term(dg[2], xa.z), term(dg[3], xa.w));
      float t2 = __fadd_rn(term(dg[4], xb.x), term(dg[5], xb.y));
      float t3 = __fadd_rn(term(dg[6], xb.z), term(dg[7], xb.w));
      float v = __fadd_rn(__fadd_rn(t0, t1), __fadd_rn(t2, t3));
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
      acc = __fadd_rn(acc, __fmul_rn(scales[r * nb + b], v));
    }
    if (lane == 0) out[j * rows + r] = acc;
  }
}

}  // namespace tr

using namespace tr;

extern "C" int tr_gemm_exact(int fmt, const uint8_t* payload, const float* scales, const float* x, float* out,
                             int64_t rows, int64_t nb, int64_t batch, int64_t row0, int64_t row1, void* stream) {
  TR_REQUIRE(fmt == kFmtTq2 || fmt == kFmtTq1, "tr_gemm_exact: bad fmt %d", fmt);
  TR_REQUIRE(0 <= row0 && row0 <= row1 && row1 <= rows && nb >= 0 && batch >= 0, "tr_gemm_exact: bad ranges");
  TR_REQUIRE(((uintptr_t)x & 15) == 0, "tr_gemm_exact: x must be 16-byte aligned");
  int64_t items = (row1 - row0) * batch;
  if (items == 0) return 0;
  int64_t grid = ceil_div(items * 32, 256);
  if (grid > 148 * 16) grid = 148 * 16;
  cudaStream_t st = (cudaStream_t)stream;
  if (fmt == kFmtTq2)
    k_gemm_exact<kFmtTq2><<<(int)grid, 256, 0, st>>>(payload, scales, x, out, rows, nb, batch, row0, row1);
  else
    k_gemm_exact<kFmtTq1><<<(int)grid, 256, 0, st>>>(payload, scales, x, out, rows, nb, batch, row0, row1);
  return check_launch("tr_gemm_exact");
}
