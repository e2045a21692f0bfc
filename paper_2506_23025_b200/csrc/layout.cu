// Offline repacker (K1): reference PackedMatrix layout (linear.py:29-95:
// payload u8 (rows, nb, 64), scales binary16 (rows, nb)) <-> the T16 device
// layout shared by the GEMV (mma.sync) and GEMM (tcgen05) kernels; bit-exact
// and invertible (tr_unrepack).  See common.cuh for the layout definition.
#include "common.cuh"

namespace tr {

// Chunk encoding E (see common.cuh): the digit of chunk column col (0..63)
// lives in word w = 2*(col>>5) + ((col>>1)&1) at bit 16*(col&1) + 8*((col>>4)&1)
// + 2*((col>>2)&3).  Every mma.m16n8k16 of the GEMV then takes its four A
// registers from one bit-field position (hb, j) of four words, so one AND per
// half2 yields values d * 4^j in a single scale class per accumulator.
__host__ __device__ inline int e_word(int col) { return 2 * (col >> 5) + ((col >> 1) & 1); }
__host__ __device__ inline int e_bit(int col) { return 16 * (col & 1) + 8 * ((col >> 4) & 1) + 2 * ((col >> 2) & 3); }

// Source of a (row, block): payload bytes at payload + (row nb + b) pstride, binary16 scale at
// sbase + (row nb + b) sstride.  PackedMatrix arrays: pstride 64|52, separate scales (sstride 2);
// TPK1 records (container.py:73-82): pstride 66|54 with the scale right after the payload.
struct RepackSrc {
  const uint8_t* payload;
  int64_t pstride;
  const uint8_t* sbase;
  int64_t sstride;
  __device__ __forceinline__ const uint8_t* pay(int64_t rb) const { return payload + rb * pstride; }
  __device__ __forceinline__ __half scale(int64_t rb) const {
    const uint8_t* p = sbase + rb * sstride;   // 2-byte aligned in both layouts
    return __ushort_as_half(*reinterpret_cast<const uint16_t*>(p));
  }
};

// One thread per output 32-bit word (256 words of payload per unit).
__global__ void k_repack_tq2(const RepackSrc src, int64_t rows, int64_t nb, int64_t n_tiles, uint8_t* __restrict__ dst) {
  const int64_t total = nb * n_tiles * 256;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tb = w >> 8;                 // unit index = t * nb + b
    const int64_t t = tb / nb, b = tb % nb;
    uint8_t* unit = dst + tb * kUnitBytes;
    const int u = (int)((w >> 2) & 63), i = (int)(w & 3);
    const int half = u >> 5, c = (u >> 3) & 3, g = (u & 7) ^ (2 * c);   // u = t16_word(half, c, g)
    const int64_t row = 16 * t + 8 * half + g;
    uint32_t word = 0;
    if (row < rows) {
      // reference chunk: 16 bytes, column col at byte col/4 bits 2*(col%4) (_kernels.pyx:23-35)
      const uint8_t* cp = src.pay(row * nb + b) + 16 * c;
      uint32_t v[4];
      if ((src.pstride & 15) == 0) {
        const uint4 v4 = *reinterpret_cast<const uint4*>(cp);
        v[0] = v4.x, v[1] = v4.y, v[2] = v4.z, v[3] = v4.w;
      } else {   // TPK1 records: 66-byte stride, 2-byte aligned
        const uint16_t* h = reinterpret_cast<const uint16_t*>(cp);
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = (uint32_t)h[2 * k] | ((uint32_t)h[2 * k + 1] << 16);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int hb = 0; hb < 2; ++hb)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int col = 32 * (i >> 1) + 16 * hb + 4 * j + 2 * (i & 1) + h;
            word |= ((v[col >> 4] >> (2 * (col & 15))) & 3u) << (16 * h + 8 * hb + 2 * j);
          }
    } else {
      word = 0x55555555u;   // digit 1 everywhere (zero trits) in padded rows
    }
    reinterpret_cast<uint32_t*>(unit)[w & 255] = word;
    if ((w & 255) < 8) {   // the 8 half2 scale pairs of this unit
      const int gg = (int)(w & 255);
      const int64_t r0 = 16 * t + gg, r1 = r0 + 8;
      const __half s0 = r0 < rows ? src.scale(r0 * nb + b) : __ushort_as_half(0);
      const __half s1 = r1 < rows ? src.scale(r1 * nb + b) : __ushort_as_half(0);
      reinterpret_cast<__half2*>(unit + kTileBlockBytes)[gg] = __halves2half2(s0, s1);
    }
  }
}

// Inverse: one thread per reference payload word (4 bytes = 16 columns).
__global__ void k_unrepack_tq2(const uint8_t* __restrict__ src, int64_t rows, int64_t nb, int64_t n_tiles,
                               uint8_t* __restrict__ payload, __half* __restrict__ scales) {
  const int64_t total = rows * nb * 16;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = q / (nb * 16), rem = q % (nb * 16), b = rem / 16;
    const int k = (int)(rem % 16), c = k >> 2, kq = k & 3;   // payload bytes 4k..4k+3 = chunk c cols 16kq..+15
    const int64_t t = row / 16;
    const int rt = (int)(row % 16), half = rt >> 3, g = rt & 7;
    const int u = t16_word(half, c, g);
    const uint8_t* unit = src + (t * nb + b) * kUnitBytes;
    const uint4 w4 = *reinterpret_cast<const uint4*>(unit + u * 16);
    const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
    uint32_t v = 0;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int col = 16 * kq + m;
      v |= ((wv[e_word(col)] >> e_bit(col)) & 3u) << (2 * m);
    }
    *reinterpret_cast<uint32_t*>(payload + (row * nb + b) * kTq2Payload + 4 * k) = v;
    if (k == 0) {
      __half2 p = reinterpret_cast<const __half2*>(unit + kTileBlockBytes)[g];
      scales[row * nb + b] = half ? __high2half(p) : __low2half(p);
    }
  }
}

// ---- TQ1 <-> T16-Q1 -----------------------------------------------------------------
__device__ __forceinline__ uint8_t enc5(const uint8_t* d, int stride) {   // codec.py:180-200
  uint32_t n = 0;
#pragma unroll
  for (int j = 0; j < 5; ++j) n = n * 3u + d[j * stride];
  return (uint8_t)((n * 256u + 242u) / 243u);
}
__device__ __forceinline__ void dec5(uint32_t s, uint8_t* d, int stride) {   // Algorithm 1
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const uint32_t p = s * 3u;
    d[j * stride] = (uint8_t)(p >> 8);
    s = p & 0xFFu;
  }
}

// one thread per (padded row, block): reference codes -> digits -> pair-group codes
__global__ void k_repack_tq1(const RepackSrc srcs, int64_t rows, int64_t nb, int64_t rows_pad,
                             uint8_t* __restrict__ dst) {
  const int64_t total = rows_pad * nb;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = q / nb, b = q % nb, t = row / 16;
    const int rt = (int)(row % 16);
    uint8_t d[260];
    if (row < rows) {
      const uint8_t* src = srcs.pay(row * nb + b);
      for (int c = 0; c < kTq1Payload; ++c) dec5(src[c], d + 5 * c, 1);
    } else {
      for (int i = 0; i < 260; ++i) d[i] = 1;
    }
    for (int i = 256; i < 260; ++i) d[i] = 1;   // pad digits (blocks.py:154-158)
    uint8_t* unit = dst + (t * nb + b) * kQ1UnitBytes;
    uint8_t* out = unit + rt * kQ1RowBytes;
    for (int g = 0; g < 26; ++g) {
      uint8_t ev[5], od[5];
      for (int k = 0; k < 5; ++k) {
        const int ce = 10 * g + 2 * k, co = ce + 1;
        ev[k] = ce < 256 ? d[ce] : 1;
        od[k] = co < 256 ? d[co] : 1;
      }
      out[2 * g] = enc5(ev, 1);
      out[2 * g + 1] = enc5(od, 1);
    }
    const __half s = row < rows ? srcs.scale(row * nb + b) : __ushort_as_half(0);
    reinterpret_cast<__half*>(unit + kQ1TileBlockBytes)[2 * (rt & 7) + (rt >> 3)] = s;
  }
}

// inverse: one thread per (row, block): pair-group codes -> digits -> reference codes
__global__ void k_unrepack_tq1(const uint8_t* __restrict__ src, int64_t rows, int64_t nb,
                               uint8_t* __restrict__ payload, __half* __restrict__ scales) {
  const int64_t total = rows * nb;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = q / nb, b = q % nb, t = row / 16;
    const int rt = (int)(row % 16);
    const uint8_t* unit = src + (t * nb + b) * kQ1UnitBytes;
    const uint8_t* in = unit + rt * kQ1RowBytes;
    uint8_t d[260];
    for (int g = 0; g < 26; ++g) {
      uint8_t ev[5], od[5];
      dec5(in[2 * g], ev, 1);
      dec5(in[2 * g + 1], od, 1);
      for (int k = 0; k < 5; ++k) {
        d[10 * g + 2 * k] = ev[k];
        d[10 * g + 2 * k + 1] = od[k];
      }
    }
    for (int i = 256; i < 260; ++i) d[i] = 1;
    uint8_t* out = payload + (row * nb + b) * kTq1Payload;
    for (int c = 0; c < kTq1Payload; ++c) out[c] = enc5(d + 5 * c, 1);
    scales[row * nb + b] = reinterpret_cast<const __half*>(unit + kQ1TileBlockBytes)[2 * (rt & 7) + (rt >> 3)];
  }
}

}  // namespace tr

using namespace tr;

extern "C" {

int64_t tr_layout_bytes(int fmt, int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1) return -1;
  int64_t nb = ceil_div(cols, kBlock), n_tiles = rows_padded(rows) / 16;
  if (fmt == kFmtTq2) return nb * n_tiles * kUnitBytes;
  if (fmt == kFmtTq1) return nb * n_tiles * kQ1UnitBytes;
  return -1;
}

static int repack_from(int fmt, const RepackSrc& src, int64_t rows, int64_t cols, void* dst, size_t dst_bytes,
                       cudaStream_t st, const char* what) {
  TR_REQUIRE(fmt == kFmtTq2 || fmt == kFmtTq1, "%s: fmt must be TQ2 (2) or TQ1 (3), got %d", what, fmt);
  TR_REQUIRE(rows >= 1 && cols >= 1, "%s: matrix must be non-empty", what);
  TR_REQUIRE(dst_bytes >= (size_t)tr_layout_bytes(fmt, rows, cols), "%s: dst holds %zu bytes, the layout needs %lld",
             what, dst_bytes, (long long)tr_layout_bytes(fmt, rows, cols));
  TR_REQUIRE(((uintptr_t)dst & 15) == 0 && ((uintptr_t)src.sbase & 1) == 0, "%s: misaligned buffers", what);
  const int64_t nb = ceil_div(cols, kBlock);
  if (fmt == kFmtTq1) {
    const int64_t rp = rows_padded(rows);
    const int grid = (int)(ceil_div(rp * nb, 128) > 148 * 32 ? 148 * 32 : ceil_div(rp * nb, 128));
    k_repack_tq1<<<grid, 128, 0, st>>>(src, rows, nb, rp, (uint8_t*)dst);
    return check_launch(what);
  }
  TR_REQUIRE(((uintptr_t)src.payload & 1) == 0 && ((src.pstride & 15) != 0 || ((uintptr_t)src.payload & 15) == 0),
             "%s: misaligned payload", what);
  const int64_t n_tiles = rows_padded(rows) / 16, total = nb * n_tiles * 256;
  const int grid = (int)(ceil_div(total, 256) > 148 * 64 ? 148 * 64 : ceil_div(total, 256));
  k_repack_tq2<<<grid, 256, 0, st>>>(src, rows, nb, n_tiles, (uint8_t*)dst);
  return check_launch(what);
}

int tr_repack(int fmt, const uint8_t* payload, const uint16_t* scales_f16, int64_t rows, int64_t cols, void* dst,
              size_t dst_bytes, void* stream) {
  const RepackSrc src = {payload, fmt == kFmtTq1 ? kTq1Payload : kTq2Payload, (const uint8_t*)scales_f16, 2};
  return repack_from(fmt, src, rows, cols, dst, dst_bytes, (cudaStream_t)stream, "tr_repack");
}

int tr_repack_records(int fmt, const uint8_t* records, int64_t rows, int64_t cols, void* dst, size_t dst_bytes,
                      void* stream) {
  const int64_t pb = fmt == kFmtTq1 ? kTq1Payload : kTq2Payload;
  const RepackSrc src = {records, pb + 2, records + pb, pb + 2};
  return repack_from(fmt, src, rows, cols, dst, dst_bytes, (cudaStream_t)stream, "tr_repack_records");
}

int tr_unrepack(int fmt, const void* src, int64_t rows, int64_t cols, size_t src_bytes, uint8_t* payload,
                uint16_t* scales_f16, void* stream) {
  TR_REQUIRE(fmt == kFmtTq2 || fmt == kFmtTq1, "tr_unrepack: fmt must be TQ2 (2) or TQ1 (3), got %d", fmt);
  TR_REQUIRE(rows >= 1 && cols >= 1, "tr_unrepack: matrix must be non-empty");
  TR_REQUIRE(src_bytes >= (size_t)tr_layout_bytes(fmt, rows, cols), "tr_unrepack: src holds %zu bytes, the layout "
             "needs %lld", src_bytes, (long long)tr_layout_bytes(fmt, rows, cols));
  if (fmt == kFmtTq1) {
    const int64_t nb = ceil_div(cols, kBlock);
    const int grid = (int)(ceil_div(rows * nb, 128) > 148 * 32 ? 148 * 32 : ceil_div(rows * nb, 128));
    k_unrepack_tq1<<<grid, 128, 0, (cudaStream_t)stream>>>((const uint8_t*)src, rows, nb, payload,
                                                           (__half*)scales_f16);
    return check_launch("tr_unrepack(tq1)");
  }
  int64_t nb = ceil_div(cols, kBlock), n_tiles = rows_padded(rows) / 16;
  int64_t total = rows * nb * 16;
  int grid = (int)(ceil_div(total, 256) > 148 * 64 ? 148 * 64 : ceil_div(total, 256));
  k_unrepack_tq2<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint8_t*)src, rows, nb, n_tiles, payload,
                                                         (__half*)scales_f16);
  return check_launch("tr_unrepack");
}

}  // extern "C"
