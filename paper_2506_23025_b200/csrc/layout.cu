// Offline repacker (K1): reference PackedMatrix layout (linear.py:29-95:
// payload u8 (rows, nb, 64), scales binary16 (rows, nb)) <-> the T16 device
// layout shared by the GEMV (mma.sync) and GEMM (tcgen05) kernels; bit-exact
// and invertible (tr_unrepack).  See common.cuh for the layout definition.
#include "common.cuh"

namespace tr {

// Chunk encoding E: digit of chunk column m (0..63) lives in word m/16 at bit
// position pos(m%16) where m%16 = 8*hb + 2*j + h  ->  pos = 16*h + 8*hb + 2*j.
__host__ __device__ inline int e_bitpos(int m16) {
  int h = m16 & 1, j = (m16 >> 1) & 3, hb = m16 >> 3;
  return 16 * h + 8 * hb + 2 * j;
}

// One thread per output 32-bit word.  Words per tile-block: 64 units x 4.
__global__ void k_repack_tq2(const uint8_t* __restrict__ payload, const __half* __restrict__ scales,
                             int64_t rows, int64_t nb, int64_t n_tiles, uint32_t* __restrict__ dst_words,
                             __half2* __restrict__ dst_scales) {
  const int64_t total = nb * n_tiles * 256;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tb = w >> 8;                 // tile-block index = b * n_tiles + t
    const int64_t b = tb / n_tiles, t = tb % n_tiles;
    const int u = (int)((w >> 2) & 63), i = (int)(w & 3);
    const int half = u >> 5, c = (u >> 3) & 3, g = u & 7;
    const int64_t row = 16 * t + 8 * half + g;
    uint32_t word = 0;
    if (row < rows) {
      const uint8_t* src = payload + (row * nb + b) * kTq2Payload + 16 * c + 4 * i;   // chunk cols 16i..16i+15
      uint32_t v = *reinterpret_cast<const uint32_t*>(src);                           // col 16i+m at bits 2m
#pragma unroll
      for (int m = 0; m < 16; ++m) word |= ((v >> (2 * m)) & 3u) << e_bitpos(m);
    } else {
      word = 0x55555555u;   // digit 1 everywhere (zero trits) in padded rows
    }
    dst_words[w] = word;
    if (u == 0 && i == 0) {
      // the 8 half2 scale pairs of this tile-block
      for (int gg = 0; gg < 8; ++gg) {
        int64_t r0 = 16 * t + gg, r1 = r0 + 8;
        __half s0 = r0 < rows ? scales[r0 * nb + b] : __ushort_as_half(0);
        __half s1 = r1 < rows ? scales[r1 * nb + b] : __ushort_as_half(0);
        dst_scales[tb * 8 + gg] = __halves2half2(s0, s1);
      }
    }
  }
}

// Inverse: one thread per reference payload word (4 bytes = 16 columns).
__global__ void k_unrepack_tq2(const uint32_t* __restrict__ src_words, const __half2* __restrict__ src_scales,
                               int64_t rows, int64_t nb, int64_t n_tiles, uint8_t* __restrict__ payload,
                               __half* __restrict__ scales) {
  const int64_t total = rows * nb * 16;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = q / (nb * 16), rem = q % (nb * 16), b = rem / 16;
    const int k = (int)(rem % 16), c = k >> 2, i = k & 3;   // payload bytes 4k..4k+3 = chunk c word i
    const int64_t t = row / 16;
    const int rt = (int)(row % 16), half = rt >> 3, g = rt & 7;
    const int u = half * 32 + c * 8 + g;
    uint32_t word = src_words[((b * n_tiles + t) * 64 + u) * 4 + i];
    uint32_t v = 0;
#pragma unroll
    for (int m = 0; m < 16; ++m) v |= ((word >> e_bitpos(m)) & 3u) << (2 * m);
    *reinterpret_cast<uint32_t*>(payload + (row * nb + b) * kTq2Payload + 4 * k) = v;
    if (k == 0) {
      __half2 p = src_scales[(b * n_tiles + t) * 8 + g];
      scales[row * nb + b] = half ? __high2half(p) : __low2half(p);
    }
  }
}

}  // namespace tr

using namespace tr;

extern "C" {

int64_t tr_layout_bytes(int fmt, int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1) return -1;
  int64_t nb = ceil_div(cols, kBlock), n_tiles = rows_padded(rows) / 16;
  if (fmt == kFmtTq2) return nb * n_tiles * (kTileBlockBytes + kTileScaleBytes);
  return -1;
}

int tr_repack(int fmt, const uint8_t* payload, const uint16_t* scales_f16, int64_t rows, int64_t cols, void* dst,
              void* stream) {
  TR_REQUIRE(fmt == kFmtTq2, "tr_repack: only TQ2 (2) uses the T16 layout, got fmt %d", fmt);
  TR_REQUIRE(rows >= 1 && cols >= 1, "tr_repack: matrix must be non-empty");
  TR_REQUIRE(((uintptr_t)payload & 3) == 0 && ((uintptr_t)dst & 15) == 0, "tr_repack: misaligned buffers");
  int64_t nb = ceil_div(cols, kBlock), n_tiles = rows_padded(rows) / 16;
  uint32_t* words = (uint32_t*)dst;
  __half2* sc = (__half2*)((uint8_t*)dst + nb * n_tiles * kTileBlockBytes);
  int64_t total = nb * n_tiles * 256;
  int grid = (int)(ceil_div(total, 256) > 148 * 64 ? 148 * 64 : ceil_div(total, 256));
  k_repack_tq2<<<grid, 256, 0, (cudaStream_t)stream>>>(payload, (const __half*)scales_f16, rows, nb, n_tiles, words, sc);
  return check_launch("tr_repack");
}

int tr_unrepack(int fmt, const void* src, int64_t rows, int64_t cols, uint8_t* payload, uint16_t* scales_f16,
                void* stream) {
  TR_REQUIRE(fmt == kFmtTq2, "tr_unrepack: only TQ2 (2) uses the T16 layout, got fmt %d", fmt);
  TR_REQUIRE(rows >= 1 && cols >= 1, "tr_unrepack: matrix must be non-empty");
  int64_t nb = ceil_div(cols, kBlock), n_tiles = rows_padded(rows) / 16;
  const uint32_t* words = (const uint32_t*)src;
  const __half2* sc = (const __half2*)((const uint8_t*)src + nb * n_tiles * kTileBlockBytes);
  int64_t total = rows * nb * 16;
  int grid = (int)(ceil_div(total, 256) > 148 * 64 ? 148 * 64 : ceil_div(total, 256));
  k_unrepack_tq2<<<grid, 256, 0, (cudaStream_t)stream>>>(words, sc, rows, nb, n_tiles, payload, (__half*)scales_f16);
  return check_launch("tr_unrepack");
}

}  // extern "C"
