// Shared device code of the int8-slice GEMV (K3-S8, gemv_s8.cu) and its persistent
// chain form (K6, gemv_chain.cu): activation staging onto the integer grid, the
// staged-slice layout and the u8 x s8 mma.sync wrappers.  See gemv_s8.cu for the method.
#pragma once

#include "common.cuh"

namespace tr {

constexpr int kS8SU = 2;
#ifndef S8_PRE1_UNITS
#define S8_PRE1_UNITS 5   // per-warp units from which only one ring slot goes out before the wait
#endif
#ifndef S8_TWO_CHAINS
#define S8_TWO_CHAINS 0   // 1: each unit's 8 IMMAs as two accumulator chains (measured 1-2% slower)
#endif              // units per ring slot (one bulk copy)
constexpr int kS8NSMax = 4;
constexpr int kS8ItemBytes = 1024;    // staged x per (block, batch row): 4 slices x 4 chunks x 16 words

template <int NW, int NG = 1> struct S8Cfg {   // NG MMA groups of 2 batch rows
  static constexpr int kSlotBytes = kS8SU * kUnitBytes;
  static constexpr size_t kRedOff = 1024;                         // [mbarriers | slot tags]
  static constexpr size_t kRedBytes = (size_t)2 * NW * 64 * NG * 4;   // 2 parked tiles per warp x 64 NG floats
  static constexpr size_t kCsOff = kRedOff + kRedBytes;           // -Cs: nb x nrx x 4 int32
  __host__ __device__ static size_t f_off(int nb, int nrx) { return kCsOff + (size_t)nb * nrx * 16; }
  __host__ __device__ static size_t xs_off(int nb, int nrx) {
    return (f_off(nb, nrx) + (size_t)nb * nrx * 4 + 127) / 128 * 128;
  }
  __host__ __device__ static size_t ring_off(int nb, int nrx) {
    return xs_off(nb, nrx) + (size_t)nb * nrx * kS8ItemBytes;
  }
  __host__ __device__ static size_t smem(int nb, int nrx, int ns) {
    return ring_off(nb, nrx) + (size_t)NW * ns * kSlotBytes;
  }
};

// Staged slice word of (block kb, batch row br, slice s, chunk c, combo cb = 4w + j): the
// 4 bytes B[k-slots] of one MMA B-fragment register.  The 16-byte group index is XOR-swizzled
// by (chunk pair, slice parity) so a quarter-warp's 128-bit loads hit 8 distinct bank groups.
__device__ __forceinline__ uint32_t s8_word_off(int nrx, int kb, int br, int s, int c, int cb) {
  const int sw = ((c >> 1) << 1) | (s & 1);
  return (uint32_t)(kb * nrx + br) * kS8ItemBytes + s * 256 + c * 64 + (((cb >> 2) ^ sw) << 4) + ((cb & 3) << 2);
}

template <typename T>
__device__ __forceinline__ void s8_f8(const uint4& v, float (&f)[8]) {
  const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = Act<T>::to_float(e[i]);
}
template <typename T>
__device__ __forceinline__ uint4 s8_pack8(const float (&f)[8]) {
  uint4 v;
  T* e = reinterpret_cast<T*>(&v);
#pragma unroll
  for (int i = 0; i < 8; ++i) e[i] = Act<T>::from_float(f[i]);
  return v;
}
template <typename T>
__device__ __forceinline__ float s8_rnd(float v) { return Act<T>::to_float(Act<T>::from_float(v)); }

template <typename T>
__device__ __noinline__ uint4 s8_load8_slow(const T* row, int64_t k, int cols) {   // ragged / unaligned rows
  T tmp[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) tmp[e] = (k + e < cols) ? row[k + e] : Act<T>::from_float(0.0f);
  return *reinterpret_cast<uint4*>(tmp);
}
// 8 activations through L2 only (ld.global.cg): for data another CTA of the same launch wrote
// (the persistent chain), where the non-coherent path could return a stale L1 line
template <typename T>
__device__ __noinline__ uint4 s8_load8_cg_slow(const T* row, int64_t k, int cols) {
  T tmp[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) tmp[e] = (k + e < cols) ? __ldcg(row + k + e) : Act<T>::from_float(0.0f);
  return *reinterpret_cast<uint4*>(tmp);
}
template <typename T>
__device__ __forceinline__ uint4 s8_load8_cg(const T* row, int64_t k, int cols, int vec) {
  if (vec && k + 8 <= cols) return __ldcg(reinterpret_cast<const uint4*>(row + k));
  return s8_load8_cg_slow(row, k, cols);
}
template <typename T>
__device__ __forceinline__ uint4 s8_load8(const T* row, int64_t k, int cols, int vec) {
  if (vec && k + 8 <= cols) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(row + k));
    return r;
  }
  return s8_load8_slow(row, k, cols);
}

// Whole warp: lane l holds the activations of columns kb*256 + 8l .. +7 of batch row br (already
// rounded to T).  Puts the block on its integer grid, stores the 4 slices in k-slot order, and
// -Cs and the block grid factor 2^(e-29).
// NI blocks at once (independent latency chains interleave); items >= nvalid are computed
// but not stored (nvalid is warp-uniform).
template <int NI>
__device__ __forceinline__ void s8_stage_blocks(const float (&f)[NI][8], uint8_t* xs, int32_t* ncs, float* fsc,
                                                int nrx, const int (&kb)[NI], const int (&br)[NI], int nvalid) {
  const int lane = threadIdx.x & 31;
  const int c = lane >> 3, mm = lane & 7;
  int ex[NI];
#pragma unroll
  for (int t = 0; t < NI; ++t) {
    float m = 0.0f;
#pragma unroll
    for (int e = 0; e < 8; ++e) m = fmaxf(m, fabsf(f[t][e]));
    const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(m));   // |x| >= 0: bits order as floats
    ex[t] = (int)((mb >> 23) & 0xFF) - 127;              // 2^ex <= max|x| < 2^(ex+1)
    ex[t] = ex[t] < -90 ? -90 : ex[t];                   // zero / tiny blocks: any grid is exact enough
  }
  // columns 8mm + e: field class j = (2mm + (e >> 2)) & 3; X = rint(x * 2^(23-ex) * 4^(3-j)), |X| <= 2^30
  uint32_t R[NI][4][2];   // [item][slice][e >> 2]: the signed-byte slices of columns e = 4G .. 4G+3
  int wj[2];
#pragma unroll
  for (int G = 0; G < 2; ++G) {
    const int j = (2 * mm + G) & 3;
    wj[G] = (1 << (2 * j)) * 0x01010101;
#pragma unroll
    for (int t = 0; t < NI; ++t) {
      const float q = __int_as_float((150 - ex[t] + 2 * (3 - j)) << 23);
      uint32_t Z[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // balanced base-256 digits: the bytes of (X + 0x80808080) ^ 0x80808080 are int8 slices of X
        Z[i] = ((uint32_t)__float2int_rn(f[t][4 * G + i] * q) + 0x80808080u) ^ 0x80808080u;
      }
      const uint32_t t0 = __byte_perm(Z[0], Z[1], 0x5140), t1 = __byte_perm(Z[0], Z[1], 0x7362);
      const uint32_t t2 = __byte_perm(Z[2], Z[3], 0x5140), t3 = __byte_perm(Z[2], Z[3], 0x7362);
      R[t][0][G] = __byte_perm(t0, t2, 0x5410);
      R[t][1][G] = __byte_perm(t0, t2, 0x7632);
      R[t][2][G] = __byte_perm(t1, t3, 0x5410);
      R[t][3][G] = __byte_perm(t1, t3, 0x7632);
    }
  }
  int cs[NI][4];
#pragma unroll
  for (int t = 0; t < NI; ++t)
#pragma unroll
    for (int s = 0; s < 4; ++s) cs[t][s] = __dp4a((int)R[t][s][1], wj[1], __dp4a((int)R[t][s][0], wj[0], 0));
  // word (s, combo) = bytes {(h0,hb0), (h0,hb1), (h1,hb0), (h1,hb1)}: columns 16 apart sit in
  // lanes 2 apart; the hb = 0 lane builds pairs 0-1, its partner pairs 2-3
  const int hb = (mm >> 1) & 1;
#pragma unroll
  for (int t = 0; t < NI; ++t)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint32_t send = hb ? R[t][s][0] : R[t][s][1];
      const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, 2);
      const uint32_t mine = hb ? R[t][s][1] : R[t][s][0];
      const uint32_t lo = hb ? recv : mine, hi = hb ? mine : recv;
#pragma unroll
      for (int pl = 0; pl < 2; ++pl) {
        const int p = pl + 2 * hb;
        const int w = 2 * (mm >> 2) + (p & 1), j = (2 * mm + (p >> 1)) & 3;
        const uint32_t word = __byte_perm(lo, hi, pl ? 0x7362 : 0x5140);
        if (t < nvalid) *reinterpret_cast<uint32_t*>(xs + s8_word_off(nrx, kb[t], br[t], s, c, 4 * w + j)) = word;
      }
    }
#pragma unroll
  for (int t = 0; t < NI; ++t)
#pragma unroll
    for (int s = 0; s < 4; ++s) cs[t][s] = __reduce_add_sync(0xffffffffu, cs[t][s]);
  if (lane == 0)
#pragma unroll
    for (int t = 0; t < NI; ++t)
      if (t < nvalid) {
        int4 v = make_int4(-cs[t][0], -cs[t][1], -cs[t][2], -cs[t][3]);
        *reinterpret_cast<int4*>(ncs + (kb[t] * nrx + br[t]) * 4) = v;
        fsc[kb[t] * nrx + br[t]] = __int_as_float((127 + ex[t] - 29) << 23);   // 2^(ex - 29)
      }
}
__device__ __forceinline__ void s8_stage_block(const float (&f)[8], uint8_t* xs, int32_t* ncs, float* fsc, int nrx,
                                               int kb, int br) {
  const float(&f1)[1][8] = *reinterpret_cast<const float(*)[1][8]>(&f);
  const int k1[1] = {kb}, b1[1] = {br};
  s8_stage_blocks<1>(f1, xs, ncs, fsc, nrx, k1, b1, 1);
}

__device__ __forceinline__ void imma(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// D = A B + C with C in separate registers (the first MMA of a chain starts from -Cs or 0)
__device__ __forceinline__ void imma_c(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1, int c0, int c1,
                                       int c2, int c3) {
  asm(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};\n"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c0), "r"(c1), "r"(c2), "r"(c3));
}
__device__ __forceinline__ uint32_t u4c(const uint4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }


}  // namespace tr
