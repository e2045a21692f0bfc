// Shared device code of the int8-slice GEMV (K3-S8, gemv_s8.cu) and its persistent
// chain form (K6, gemv_chain.cu): activation staging onto the integer grid, the
// staged-slice layout and the u8 x s8 mma.sync wrappers.  See gemv_s8.cu for the method.
#pragma once

#include "common.cuh"

namespace tr {

constexpr int kS8SU = 2;
#ifndef S8_PRE1_UNITS
#define S8_PRE1_UNITS 4   // per-warp units from which only one ring slot goes out before the wait (re-measured: 4 over 5, +0.3%)
#endif
#ifndef S8_TWO_CHAINS
#define S8_TWO_CHAINS 0   // 1: each unit's 8 IMMAs as two accumulator chains (measured 1-2% slower)
#endif              // units per ring slot (one bulk copy)
#ifndef S8_NS_MAX
#define S8_NS_MAX 4
#endif
constexpr int kS8NSMax = S8_NS_MAX;
constexpr int kS8ItemBytes = 1024;    // staged x per (block, batch row): 4 slices x 4 chunks x 16 words
constexpr int kQ1ItemBytes = 1280;    // TQ1: 4 slices x 4 lane columns x 80 B (18 words of 9 MMAs + pad)

template <int FMT> struct S8Fmt {      // TQ2 (T16 units) or TQ1 (T16-Q1 units)
  static constexpr int kUnit = FMT == kFmtTq1 ? kQ1UnitBytes : kUnitBytes;
  static constexpr int kItem = FMT == kFmtTq1 ? kQ1ItemBytes : kS8ItemBytes;
  static constexpr int kTileBlock = FMT == kFmtTq1 ? kQ1TileBlockBytes : kTileBlockBytes;
};

template <int NW, int NG = 1, int FMT = kFmtTq2> struct S8Cfg {   // NG MMA groups of 2 batch rows
  static constexpr int kSlotBytes = kS8SU * S8Fmt<FMT>::kUnit;
  static constexpr size_t kRedOff = 1024;                         // [mbarriers | slot tags]
  static constexpr size_t kRedBytes = (size_t)2 * NW * 64 * NG * 4;   // 2 parked tiles per warp x 64 NG floats
  static constexpr size_t kCsOff = kRedOff + kRedBytes;           // -Cs: nb x nrx x 4 int32
  __host__ __device__ static size_t f_off(int nb, int nrx) { return kCsOff + (size_t)nb * nrx * 16; }
  __host__ __device__ static size_t xs_off(int nb, int nrx) {
    return (f_off(nb, nrx) + (size_t)nb * nrx * 4 + 127) / 128 * 128;
  }
  __host__ __device__ static size_t ring_off(int nb, int nrx) {
    return xs_off(nb, nrx) + (size_t)nb * nrx * S8Fmt<FMT>::kItem;
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


// ---- K4: the TQ1 (1.6 bit) GEMV on the same int8 tensor-core path ----------------------------
//
// T16-Q1 rows hold 26 pair-groups (A_g, B_g): base-3 codes of columns 10g + {0,2,4,6,8} and
// 10g + {1,3,5,7,9} (common.cuh).  Algorithm 1 (reference _kernels.pyx:73-87)
// gives digit k (k = 1..5) of code c as d_k = F_k - 3 F_{k-1}, F_k = floor(3^k c / 256), F_0 = 0
// (s_k = 3^k c mod 256 by induction, and 3^k c = 768 F_{k-1} + 3 s_{k-1}).  Summation by parts
// moves the subtraction onto the activations:
//     sum_k d_k x_k = sum_k F_k (x_k - 3 x_{k+1}),   x_6 := 0,
// with x_k the activation of digit k's column.  F_k <= 242 is a u8 MMA operand, and with
// R = A_g | B_g << 16 one IMAD R * 3^k yields F_k of both codes in bytes 1 and 3 (3^5 * 255 <
// 2^16: the 16-bit lanes never carry into each other) -- 5 IMADs per 10 weights, one PRMT per 4
// MMA operand bytes, no digit extraction.  Staging turns x into B'_k = x~_k - 3 x~_{k+2 columns}
// on the integer grid (exact), sliced into int8 as in K3-S8, and the trit offset is folded as
// before: D = sum F B' - sum x~ (= sum (d - 1) x~).
//
// K-slot order.  Lane column c of the MMA fragments owns pair-groups [G0(c), G0(c) + 7) of its
// two rows, G0 = {0, 7, 14, 20} (7, 7, 6, 6 groups); result rho = 5 gl + (k - 1) of local group
// gl, packed two per A register: register m = {F(2m).A, F(2m).B, F(2m+1).A, F(2m+1).B}.  Nine
// MMAs (288 K slots) cover a row's 260 digits; slots past a lane's groups get B' = 0, so the
// bytes a lane decodes past its own groups (harmless reads inside the unit) never count.
__host__ __device__ inline int q1_g0(int c) { return c == 0 ? 0 : c == 1 ? 7 : c == 2 ? 14 : 20; }
__host__ __device__ inline int q1_ng(int c) { return c < 2 ? 7 : 6; }

// Stage one (block, batch row) item for K4 (whole warp; lane holds columns 8 lane .. + 7):
// x~ on the block's integer grid, -Cs of the x~ slices, the grid factor 2^(ex - 23), and the 288
// B' slots as int8 slices at [slice s][lane column c][word m] (80 B rows, 16-B aligned).
// Slot table of the B' staging: entry (p, b) of lane L = column | valid << 16 | has-next << 17 of byte b
// of quad lane + 32 p (lane column c' = quad / 18, register m = quad % 18).  384 ints, one pass.
__device__ __forceinline__ void s8q1_slot_table(int* tab) {
  for (int i = threadIdx.x; i < 12 * 32; i += blockDim.x) {
    const int pb = i >> 5, lane = i & 31, p = pb >> 2, b = pb & 3;
    const int qd = lane + 32 * p, cq = qd / 18, m = qd - 18 * cq;
    const int rho = 2 * m + (b >> 1), gl = rho / 5, k1 = rho - 5 * gl;
    const int col = 10 * (q1_g0(cq & 3) + gl) + 2 * k1 + (b & 1);
    const bool valid = qd < 72 && rho < 5 * q1_ng(cq & 3) && col < 256;
    const bool next = valid && k1 < 4 && col + 2 < 256;
    // byte offsets into the staging scratch (column c at word (c & 3) * 64 + (c >> 2)); 1024 is a
    // zero word, so slots without a column (or without a next digit) read 0 branch-free
    const int o1 = valid ? 4 * ((col & 3) * 64 + (col >> 2)) : 1024;
    const int o2 = next ? 4 * (((col + 2) & 3) * 64 + ((col + 2) >> 2)) : 1024;
    tab[i] = o1 | (o2 << 16);
  }
}

__device__ __forceinline__ uint32_t s8_lds32(uint32_t addr) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(r) : "r"(addr) : "memory");
  return r;
}
__device__ __forceinline__ void s8q1_stage_block(const float (&f)[8], uint8_t* item, int32_t* ncs_item,
                                                 float* fsc_item, const int* tab) {
  const int lane = threadIdx.x & 31;
  float mx = 0.0f;
#pragma unroll
  for (int e = 0; e < 8; ++e) mx = fmaxf(mx, fabsf(f[e]));
  const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
  int ex = (int)((mb >> 23) & 0xFF) - 127;
  ex = ex < -90 ? -90 : ex;
  const float q = __int_as_float((150 - ex) << 23);   // 2^(23 - ex)
  int xi[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) xi[e] = __float2int_rn(f[e] * q);
  // -Cs: per slice, the sum over the block of the balanced int8 slices of x~
  int cs[4] = {0, 0, 0, 0};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t Z[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) Z[i] = ((uint32_t)xi[4 * h + i] + 0x80808080u) ^ 0x80808080u;
    const uint32_t t0 = __byte_perm(Z[0], Z[1], 0x5140), t1 = __byte_perm(Z[0], Z[1], 0x7362);
    const uint32_t t2 = __byte_perm(Z[2], Z[3], 0x5140), t3 = __byte_perm(Z[2], Z[3], 0x7362);
    cs[0] = __dp4a((int)__byte_perm(t0, t2, 0x5410), 0x01010101, cs[0]);
    cs[1] = __dp4a((int)__byte_perm(t0, t2, 0x7632), 0x01010101, cs[1]);
    cs[2] = __dp4a((int)__byte_perm(t1, t3, 0x5410), 0x01010101, cs[2]);
    cs[3] = __dp4a((int)__byte_perm(t1, t3, 0x7632), 0x01010101, cs[3]);
  }
#pragma unroll
  for (int s = 0; s < 4; ++s) cs[s] = __reduce_add_sync(0xffffffffu, cs[s]);
  // x~ as int32 scratch in the item's own bytes, column c at word (c & 3) * 64 + (c >> 2): the slot
  // gather below reads columns ~4 apart across lanes, which this layout spreads over the banks
  // (26 shared-memory wavefronts per block instead of 62)
  int* scr = reinterpret_cast<int*>(item);
#pragma unroll
  for (int e = 0; e < 8; ++e) scr[(e & 3) * 64 + 2 * lane + (e >> 2)] = xi[e];
  if (lane == 0) scr[256] = 0;   // the zero word (item bytes 1024..1027; overwritten only after the gather)
  __syncwarp();
  const uint32_t scr32 = smem_u32(item);
  // 72 quads (lane column c', register m): four B' slots each -> one word per slice.  The slot ->
  // column map depends on the lane only: read from the table s8q1_slot_table built once per CTA.
  uint32_t W[3][4];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    uint32_t Z[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t e = (uint32_t)tab[(p * 4 + b) * 32 + lane];   // byte offsets of x~[col], x~[col + 2]
      const int x1 = (int)s8_lds32(scr32 + (e & 0xFFFFu));
      const int x2 = (int)s8_lds32(scr32 + (e >> 16));
      Z[b] = ((uint32_t)(x1 - 3 * x2) + 0x80808080u) ^ 0x80808080u;
    }
    const uint32_t t0 = __byte_perm(Z[0], Z[1], 0x5140), t1 = __byte_perm(Z[0], Z[1], 0x7362);
    const uint32_t t2 = __byte_perm(Z[2], Z[3], 0x5140), t3 = __byte_perm(Z[2], Z[3], 0x7362);
    W[p][0] = __byte_perm(t0, t2, 0x5410);
    W[p][1] = __byte_perm(t0, t2, 0x7632);
    W[p][2] = __byte_perm(t1, t3, 0x5410);
    W[p][3] = __byte_perm(t1, t3, 0x7632);
  }
  __syncwarp();   // every lane has read the scratch before the words overwrite it
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int qd = lane + 32 * p;
    if (qd < 72) {
      const int cq = qd / 18, m = qd - 18 * cq;
#pragma unroll
      for (int s = 0; s < 4; ++s) *reinterpret_cast<uint32_t*>(item + (s * 4 + cq) * 80 + m * 4) = W[p][s];
    }
  }
  if (lane == 0) {
    *reinterpret_cast<int4*>(ncs_item) = make_int4(-cs[0], -cs[1], -cs[2], -cs[3]);
    *fsc_item = __int_as_float((127 + ex - 23) << 23);   // 2^(ex - 23)
  }
}

// One T16-Q1 unit (16 rows x 256 columns) against one staged block: 9 u8 x s8 MMAs per group of
// two batch rows.  up: the unit in shared memory; xq[G2]: shared address of this lane's 18 B'
// words (slice sB, lane column c) for the block; cs: the trit offsets -Cs of its D columns.
template <int NG>
__device__ __forceinline__ void q1_unit_mma(const uint8_t* up, int g, int c, const uint32_t (&xq)[NG],
                                            const int2 (&cs)[NG], int (&D)[NG][4]) {
  const int wo = (c * 14) >> 2;   // first 32-bit word of byte 2 G0(c): 0, 3, 7, 10
  const uint32_t* r0 = reinterpret_cast<const uint32_t*>(up + kQ1RowBytes * g) + wo;
  const uint32_t* r1 = reinterpret_cast<const uint32_t*>(up + kQ1RowBytes * (g + 8)) + wo;
  uint32_t w0[5], w1[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    w0[i] = r0[i];
    w1[i] = r1[i];
  }
  const uint32_t sh = (c == 1) ? 16u : 0u;   // lane column 1 starts mid-word (byte 14)
  uint32_t R0[7], R1[7];                     // pair-group registers A_g | B_g << 16
#pragma unroll
  for (int gl = 0; gl < 7; ++gl) {
    const int i = gl >> 1;
    const uint32_t a0 = __funnelshift_r(w0[i], w0[i + 1], sh), a1 = __funnelshift_r(w1[i], w1[i + 1], sh);
    R0[gl] = __byte_perm(a0, 0u, (gl & 1) ? 0x4342 : 0x4140);
    R1[gl] = __byte_perm(a1, 0u, (gl & 1) ? 0x4342 : 0x4140);
  }
  uint32_t xb[NG][18];
#pragma unroll
  for (int G2 = 0; G2 < NG; ++G2) {
#pragma unroll
    for (int i4 = 0; i4 < 4; ++i4) {
      const uint4 v = ld_shared_v4u(xq[G2] + 16 * i4);
      xb[G2][4 * i4] = v.x;
      xb[G2][4 * i4 + 1] = v.y;
      xb[G2][4 * i4 + 2] = v.z;
      xb[G2][4 * i4 + 3] = v.w;
    }
    uint32_t lo, hi;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(lo), "=r"(hi) : "r"(xq[G2] + 64));
    xb[G2][16] = lo;
    xb[G2][17] = hi;
  }
  constexpr uint32_t kPow3[5] = {3u, 9u, 27u, 81u, 243u};
  auto res = [&](const uint32_t (&R)[7], int rho) -> uint32_t {   // F of both codes in bytes 1, 3
    return rho < 35 ? R[rho / 5] * kPow3[rho % 5] : 0u;
  };
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const uint32_t A[4] = {__byte_perm(res(R0, 4 * i), res(R0, 4 * i + 1), 0x7531),
                           __byte_perm(res(R1, 4 * i), res(R1, 4 * i + 1), 0x7531),
                           __byte_perm(res(R0, 4 * i + 2), res(R0, 4 * i + 3), 0x7531),
                           __byte_perm(res(R1, 4 * i + 2), res(R1, 4 * i + 3), 0x7531)};
#pragma unroll
    for (int G2 = 0; G2 < NG; ++G2) {
      if (i == 0)
        imma_c(D[G2], A, xb[G2][0], xb[G2][1], cs[G2].x, cs[G2].y, cs[G2].x, cs[G2].y);
      else
        imma(D[G2], A, xb[G2][2 * i], xb[G2][2 * i + 1]);
    }
  }
}

}  // namespace tr
