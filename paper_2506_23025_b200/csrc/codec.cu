// Device implementations of the reference kernel-module surface
// (tritpack/_kernels.pyx:23-133, numpy twin _kernels_py.py:46-102) and the
// fused quantize+pack used by pack_matrix (linear.py:98-120 + blocks.py:142-161).
// All are bit-exact with the reference: integer work is exact and the only
// float operations (absmax, IEEE reciprocal, one multiply, comparisons,
// fp32->fp16 RNE) are the reference's own, in the same order.
#include "common.cuh"

namespace tr {

__global__ void k_pack_base4(const uint8_t* __restrict__ d, uint8_t* __restrict__ out, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uchar4 q = reinterpret_cast<const uchar4*>(d)[i];
    out[i] = (uint8_t)(q.x | (q.y << 2) | (q.z << 4) | (q.w << 6));
  }
}

__global__ void k_unpack_base4(const uint8_t* __restrict__ w, uint8_t* __restrict__ out, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = w[i];
    reinterpret_cast<uchar4*>(out)[i] = make_uchar4(v & 3, (v >> 2) & 3, (v >> 4) & 3, (v >> 6) & 3);
  }
}

__device__ __forceinline__ uint8_t encode5(const uint8_t* d) {
  uint32_t n = d[0];
  n = n * 3u + d[1];
  n = n * 3u + d[2];
  n = n * 3u + d[3];
  n = n * 3u + d[4];
  return (uint8_t)((n * 256u + 242u) / 243u);   // codec.py:180-200 scaling, k=5 p=8
}

__global__ void k_encode_base3(const uint8_t* __restrict__ d, uint8_t* __restrict__ out, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = encode5(d + 5 * i);
}

// Algorithm 1 (_kernels.pyx:73-87): state*3, digit = high byte.
__global__ void k_decode_base3(const uint8_t* __restrict__ c, uint8_t* __restrict__ out, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t s = c[i];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      uint32_t p = s * 3u;
      out[5 * i + j] = (uint8_t)(p >> 8);
      s = p & 0xFFu;
    }
  }
}

// |x| as used by the reference absmax loop (_kernels.pyx:104-108): the max is
// taken over non-negative values starting from +0.0, so clearing the sign bit
// and comparing bit patterns as integers gives the identical float32 result.
__device__ __forceinline__ uint32_t abs_bits(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

__device__ __forceinline__ uint8_t digit_of(float v, float inv) {
  float q = __fmul_rn(v, inv);                  // float32 product, no contraction
  return q >= 0.5f ? 2 : (q <= -0.5f ? 0 : 1);  // _kernels_py.py:13-15
}

// One warp per 256-element block: lane l holds elements 8l..8l+7.
__global__ void k_quantize_blocks(const float* __restrict__ v, uint8_t* __restrict__ digits,
                                  float* __restrict__ scales, int64_t nb) {
  const int lane = threadIdx.x & 31;
  int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (; b < nb; b += nwarps) {
    const float4* src = reinterpret_cast<const float4*>(v + b * kBlock + lane * 8);
    float4 a = src[0], c = src[1];
    float e[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    uint32_t am = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) am = max(am, abs_bits(e[k]));
#pragma unroll
    for (int o = 16; o; o >>= 1) am = max(am, __shfl_xor_sync(0xffffffffu, am, o));
    float s = __uint_as_float(am);
    float inv = s > 0.0f ? 1.0f / s : 0.0f;   // IEEE div.rn (no fast-math): == float32(1) / s
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) lo |= (uint32_t)digit_of(e[k], inv) << (8 * k);
#pragma unroll
    for (int k = 0; k < 4; ++k) hi |= (uint32_t)digit_of(e[4 + k], inv) << (8 * k);
    reinterpret_cast<uint2*>(digits + b * kBlock)[lane] = make_uint2(lo, hi);
    if (lane == 0) scales[b] = s;
  }
}

__global__ void k_dequantize_blocks(const uint8_t* __restrict__ d, const float* __restrict__ s,
                                    float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fmul_rn((float)d[i] - 1.0f, s[i / kBlock]);   // _kernels.pyx:127-132
}

// pack_matrix on device: W f32 (rows, cols) -> payload (rows, nb, pb) + scales
// binary16 (rows, nb).  Columns >= cols are zero (linear.py:110-112); TQ1
// appends four pad digits of 1 (blocks.py:154-158).  One warp per (row, block).
__global__ void k_quantize_pack(const float* __restrict__ W, int64_t rows, int64_t cols, int fmt,
                                uint8_t* __restrict__ payload, __half* __restrict__ scales) {
  __shared__ uint8_t sdig[8][264];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nb = ceil_div(cols, kBlock);
  int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (; item < rows * nb; item += nwarps) {
    const int64_t r = item / nb, b = item % nb;
    const float* src = W + r * cols;
    float e[8];
    uint32_t am = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int64_t col = b * kBlock + lane * 8 + k;
      e[k] = col < cols ? src[col] : 0.0f;
      am = max(am, abs_bits(e[k]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) am = max(am, __shfl_xor_sync(0xffffffffu, am, o));
    float s = __uint_as_float(am);
    float inv = s > 0.0f ? 1.0f / s : 0.0f;
    uint8_t dg[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) dg[k] = digit_of(e[k], inv);
    if (fmt == kFmtTq2) {
      uint8_t b0 = dg[0] | (dg[1] << 2) | (dg[2] << 4) | (dg[3] << 6);
      uint8_t b1 = dg[4] | (dg[5] << 2) | (dg[6] << 4) | (dg[7] << 6);
      uint8_t* dst = payload + (r * nb + b) * kTq2Payload + lane * 2;
      dst[0] = b0;
      dst[1] = b1;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) sdig[wib][lane * 8 + k] = dg[k];
      if (lane < 4) sdig[wib][256 + lane] = 1;
      __syncwarp();
      uint8_t* dst = payload + (r * nb + b) * kTq1Payload;
      for (int c = lane; c < kTq1Payload; c += 32) dst[c] = encode5(&sdig[wib][5 * c]);
      __syncwarp();
    }
    if (lane == 0) scales[r * nb + b] = __float2half_rn(s);   // astype('<f2'): RNE
  }
}

// Dense dequantization to the activation dtype (rows, cols) for the cuBLAS
// baseline / debugging: value = f16(scale) * (d - 1), exact in fp16.
template <typename T>
__global__ void k_dequant_dense(const uint8_t* __restrict__ payload, const __half* __restrict__ scales,
                                int64_t rows, int64_t cols, int fmt, T* __restrict__ out) {
  const int64_t nb = ceil_div(cols, kBlock);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * cols; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, col = i % cols, b = col / kBlock, e = col % kBlock;
    uint32_t d;
    if (fmt == kFmtTq2) {
      d = (payload[(r * nb + b) * kTq2Payload + e / 4] >> (2 * (e % 4))) & 3;
    } else {
      uint32_t s = payload[(r * nb + b) * kTq1Payload + e / 5];
      for (int j = 0; j <= (int)(e % 5); ++j) { uint32_t p = s * 3u; d = p >> 8; s = p & 0xFFu; }
    }
    float v = __half2float(scales[r * nb + b]) * ((float)d - 1.0f);
    out[i] = Act<T>::from_float(v);
  }
}

static inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = ceil_div(n, threads);
  return (int)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

}  // namespace tr

// ---------------------------------------------------------------------------------
using namespace tr;

extern "C" {

int tr_pack_base4(const uint8_t* digits, uint8_t* words, int64_t m, void* stream) {
  TR_REQUIRE(m >= 0, "tr_pack_base4: negative length");
  if (m == 0) return 0;
  k_pack_base4<<<grid_for(m), 256, 0, (cudaStream_t)stream>>>(digits, words, m);
  return check_launch("tr_pack_base4");
}

int tr_unpack_base4(const uint8_t* words, uint8_t* digits, int64_t m, void* stream) {
  TR_REQUIRE(m >= 0, "tr_unpack_base4: negative length");
  if (m == 0) return 0;
  k_unpack_base4<<<grid_for(m), 256, 0, (cudaStream_t)stream>>>(words, digits, m);
  return check_launch("tr_unpack_base4");
}

int tr_encode_base3(const uint8_t* digits, uint8_t* codes, int64_t m, void* stream) {
  TR_REQUIRE(m >= 0, "tr_encode_base3: negative length");
  if (m == 0) return 0;
  k_encode_base3<<<grid_for(m), 256, 0, (cudaStream_t)stream>>>(digits, codes, m);
  return check_launch("tr_encode_base3");
}

int tr_decode_base3(const uint8_t* codes, uint8_t* digits, int64_t m, void* stream) {
  TR_REQUIRE(m >= 0, "tr_decode_base3: negative length");
  if (m == 0) return 0;
  k_decode_base3<<<grid_for(m), 256, 0, (cudaStream_t)stream>>>(codes, digits, m);
  return check_launch("tr_decode_base3");
}

int tr_quantize_blocks(const float* values, uint8_t* digits, float* scales, int64_t nb, void* stream) {
  TR_REQUIRE(nb >= 0, "tr_quantize_blocks: negative block count");
  TR_REQUIRE(((uintptr_t)values & 15) == 0 && ((uintptr_t)digits & 7) == 0, "tr_quantize_blocks: misaligned buffers");
  if (nb == 0) return 0;
  k_quantize_blocks<<<grid_for(nb * 32), 256, 0, (cudaStream_t)stream>>>(values, digits, scales, nb);
  return check_launch("tr_quantize_blocks");
}

int tr_dequantize_blocks(const uint8_t* digits, const float* scales, float* out, int64_t nb, void* stream) {
  TR_REQUIRE(nb >= 0, "tr_dequantize_blocks: negative block count");
  if (nb == 0) return 0;
  k_dequantize_blocks<<<grid_for(nb * kBlock), 256, 0, (cudaStream_t)stream>>>(digits, scales, out, nb * kBlock);
  return check_launch("tr_dequantize_blocks");
}

int tr_quantize_pack(int fmt, const float* W, int64_t rows, int64_t cols, uint8_t* payload,
                     uint16_t* scales_f16, void* stream) {
  TR_REQUIRE(fmt == kFmtTq2 || fmt == kFmtTq1, "tr_quantize_pack: fmt must be TQ2(2) or TQ1(3), got %d", fmt);
  TR_REQUIRE(rows >= 1 && cols >= 1, "tr_quantize_pack: matrix must be non-empty, got %lldx%lld",
             (long long)rows, (long long)cols);
  int64_t items = rows * ceil_div(cols, kBlock);
  k_quantize_pack<<<grid_for(items * 32), 256, 0, (cudaStream_t)stream>>>(W, rows, cols, fmt, payload,
                                                                          (__half*)scales_f16);
  return check_launch("tr_quantize_pack");
}

int tr_dequant_dense(int fmt, const uint8_t* payload, const uint16_t* scales_f16, int64_t rows, int64_t cols,
                     int act_dtype, void* out, void* stream) {
  TR_REQUIRE(fmt == kFmtTq2 || fmt == kFmtTq1, "tr_dequant_dense: bad fmt %d", fmt);
  TR_REQUIRE(rows >= 1 && cols >= 1, "tr_dequant_dense: empty matrix");
  cudaStream_t st = (cudaStream_t)stream;
  if (act_dtype == kActF16)
    k_dequant_dense<__half><<<grid_for(rows * cols), 256, 0, st>>>(payload, (const __half*)scales_f16, rows, cols,
                                                                   fmt, (__half*)out);
  else if (act_dtype == kActBf16)
    k_dequant_dense<__nv_bfloat16><<<grid_for(rows * cols), 256, 0, st>>>(payload, (const __half*)scales_f16, rows,
                                                                          cols, fmt, (__nv_bfloat16*)out);
  else
    TR_REQUIRE(false, "tr_dequant_dense: act_dtype must be F16(1) or BF16(2), got %d", act_dtype);
  return check_launch("tr_dequant_dense");
}

}  // extern "C"
