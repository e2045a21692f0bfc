// K5: ternary GEMM on the 5th-generation tensor cores (tcgen05 / TMEM / TMA), TQ2 weights.
//
// Semantics (reference linear.py:137-166, _kernels.pyx:136-168; paper App. F):
//   y[n, r] = sum_b s[r, b] * (sum_{k in block b} trit[r, k] * x[n, k])
// fp16/bf16 activations, fp32 accumulation, each 256-block's sum scaled by the fp32
// value of its binary16 scale; one rounding of the output.
//
// B200 design:
//  * CTA tile = 128 weight rows (8 T16 tiles) x N activation rows (N = 16..128),
//    over a K range of 256-blocks (split-K when the grid would not fill the SMs);
//  * A operand = the decoded trits, written by the CUDA cores straight into TMEM
//    (tcgen05.st), double-buffered per 256-block: per half2 one LOP3 (field | magic
//    exponent) + one HFMA2 gives trit values exactly, in natural K order;
//  * B operand = activations, loaded by TMA (128B-swizzled, K-major boxes of 64),
//    so the tensor core reads them from shared memory without any thread touching them;
//  * one elected thread issues 16 tcgen05.mma (M=128, N, K=16, A from TMEM) per
//    block into a TMEM accumulator; workers read it back (tcgen05.ld) and apply the
//    block's fp32 scale (per-block mode), or -- when every row has one scale for all
//    its blocks (per-channel gamma) -- the MMA accumulates over all K and the scale is
//    applied once;
//  * warp roles: 8 decode/epilogue warps (two per TMEM lane quadrant), 1 TMA producer
//    warp (weights by cp.async.bulk, activations by cp.async.bulk.tensor), 1 MMA warp.
//    All hand-offs are mbarriers; there is no __syncthreads in the main loop.
#include <cuda.h>

#include <type_traits>

#include "common.cuh"

namespace tr {

namespace umma {

#ifndef UMMA_TRACE
#define UMMA_TRACE 0
#endif
// CTA-0 clock trace (probe 4) compiled in only for dev builds (-DUMMA_TRACE=1): its checks sat in
// the decode and MMA loops of every launch
constexpr bool kTrace = UMMA_TRACE != 0;
#ifndef UMMA_ILV
#define UMMA_ILV 1
#endif
constexpr bool kIlv = UMMA_ILV != 0;           // uniform scale, N <= 32: warp groups decode alternate blocks
#ifndef UMMA_MERGE
#define UMMA_MERGE 1
#endif
#ifndef UMMA_ILV_MAXN
#define UMMA_ILV_MAXN 32
#endif
constexpr int kWorkers = 8;                    // decode/epilogue warps
constexpr int kThreads = (kWorkers + 2) * 32;  // + producer warp + MMA warp
constexpr int kRowsPerCta = 128;

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// The 16 MMAs of one 256-column block (A: 16 x 8 TMEM columns from a_tmem; B: the block's four
// 128B-swizzled 64-K atoms at b_smem, N rows each), issued by one elected lane in one asm block.
// The first MMA accumulates iff acc0; the rest always do.
template <int N>
__device__ __forceinline__ void mma_block16(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_smem, uint32_t idesc,
                                            int acc0) {
  // One descriptor is built from the base address inside the asm; the other 15 are that plus the
  // MMA's offset in 16-B units (the 14-bit start field cannot carry: shared addresses stay below
  // 256 KB), so ptxas keeps the whole sequence in the uniform datapath at one add per MMA.
  // Descriptor: start address (bits 0-13, 16-B units) | LBO 16 B | SBO 1024 B | version 1 |
  // 128-B swizzle.  B offset of MMA kk: (kk >> 2) * N * 128 + (kk & 3) * 32 bytes; A: kk * 8 columns.
  asm volatile(
      "{\n.reg .pred e, p;\n.reg .b32 t;\n.reg .b64 base, dd;\n"
      "shr.u32 t, %2, 4;\nand.b32 t, t, 0x3FFF;\ncvt.u64.u32 base, t;\nor.b64 base, base, 0x4000404000010000;\n"
      "elect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@!e bra SKIP_%=;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], base, %3, p;\n"
      "add.s64 dd, base, 2;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+8], dd, %3, 1;\n"
      "add.s64 dd, base, 4;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+16], dd, %3, 1;\n"
      "add.s64 dd, base, 6;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+24], dd, %3, 1;\n"
      "add.s64 dd, base, %5;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+32], dd, %3, 1;\n"
      "add.s64 dd, base, %5+2;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+40], dd, %3, 1;\n"
      "add.s64 dd, base, %5+4;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+48], dd, %3, 1;\n"
      "add.s64 dd, base, %5+6;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+56], dd, %3, 1;\n"
      "add.s64 dd, base, %6;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+64], dd, %3, 1;\n"
      "add.s64 dd, base, %6+2;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+72], dd, %3, 1;\n"
      "add.s64 dd, base, %6+4;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+80], dd, %3, 1;\n"
      "add.s64 dd, base, %6+6;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+88], dd, %3, 1;\n"
      "add.s64 dd, base, %7;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+96], dd, %3, 1;\n"
      "add.s64 dd, base, %7+2;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+104], dd, %3, 1;\n"
      "add.s64 dd, base, %7+4;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+112], dd, %3, 1;\n"
      "add.s64 dd, base, %7+6;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1+120], dd, %3, 1;\n"
      "SKIP_%=:\n}\n"
      ::"r"(d_tmem), "r"(a_tmem), "r"(b_smem), "r"(idesc), "r"(acc0), "n"(N * 8), "n"(2 * N * 8), "n"(3 * N * 8));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
               ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
        "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// 32 lanes x NC consecutive 32-bit columns -> r[NC] (NC = 8, 16 or 32); completes at tmem_wait_ld
template <int NC>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[NC]) {
  if constexpr (NC == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
  } else if constexpr (NC == 16) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                 "[%16];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15])
                 : "r"(taddr)
                 : "memory");
  } else {
    static_assert(NC == 32, "8, 16 or 32 columns");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
  }
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }


// trit decode: field (digit d at mantissa bits 2j of each half, j-class of the E layout)
// -> exact trit d - 1 as a half2 / bfloat162.  One LOP3 + one HFMA2.
template <typename T> struct Dec;
template <> struct Dec<__half> {
  static constexpr uint32_t kMagic = 0x64006400u;   // 1024.0
  __device__ static uint32_t trit2(uint32_t w, uint32_t w8, int hb, int j) {
    const uint32_t v = lop3_and_or(hb ? w8 : w, 0x00030003u << (2 * j), kMagic);   // 1024 + 4^j d
    const float m = (float)(1 << (2 * j));
    const __half2 r = __hfma2(*reinterpret_cast<const __half2*>(&v), __float2half2_rn(1.0f / m),
                              __float2half2_rn(-(1024.0f / m + 1.0f)));
    return *reinterpret_cast<const uint32_t*>(&r);
  }
};
template <> struct Dec<__nv_bfloat16> {
  static constexpr uint32_t kMagic = 0x43004300u;   // 128.0 (7 mantissa bits: fields j < 3)
  __device__ static uint32_t trit2(uint32_t w, uint32_t w8, int hb, int j) {
    uint32_t v;
    float m;
    if (j < 3) {
      v = lop3_and_or(hb ? w8 : w, 0x00030003u << (2 * j), kMagic);   // 128 + 4^j d
      m = (float)(1 << (2 * j));
    } else {
      v = lop3_and_or(w >> (hb ? 14 : 6), 0x00030003u, kMagic);        // 128 + d
      m = 1.0f;
    }
    const __nv_bfloat162 r = __hfma2(*reinterpret_cast<const __nv_bfloat162*>(&v), __float2bfloat162_rn(1.0f / m),
                                     __float2bfloat162_rn(-(128.0f / m + 1.0f)));
    return *reinterpret_cast<const uint32_t*>(&r);
  }
};

// TQ1 pair-group decode (layout in common.cuh): register A_g | B_g << 16, Algorithm-1 step
// p = 3s on both 16-bit lanes, digit at bits 8..9 of each lane -> exact trit half2 of the
// natural-order column pair (10g + 2k, 10g + 2k + 1).  Half 0 of a row writes TMEM columns
// 0..63 (groups 0..11, group 12 steps 0..3), half 1 columns 64..127 (group 12 step 4,
// groups 13..24, group 25 steps 0..2).
template <typename T> __device__ __forceinline__ uint32_t q1_trit2(uint32_t p);
template <> __device__ __forceinline__ uint32_t q1_trit2<__half>(uint32_t p) {
  const uint32_t v = lop3_and_or(p, 0x03000300u, 0x64006400u);   // 1024 + 256 d
  const __half2 r = __hfma2(*reinterpret_cast<const __half2*>(&v), __float2half2_rn(1.0f / 256.0f),
                            __float2half2_rn(-5.0f));
  return *reinterpret_cast<const uint32_t*>(&r);
}
template <> __device__ __forceinline__ uint32_t q1_trit2<__nv_bfloat16>(uint32_t p) {
  const uint32_t v = lop3_and_or(p >> 8, 0x00030003u, 0x43004300u);   // 128 + d
  const __nv_bfloat162 r = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&v), __float2bfloat162_rn(-129.0f));
  return *reinterpret_cast<const uint32_t*>(&r);
}
template <typename T, int G0, int G1, int K0LAST, int KLAST, int C0>
__device__ __forceinline__ void q1_groups(const uint32_t (&wq)[7], int wbase, uint32_t (&col)[64]) {
  // groups G0..G1 (inclusive); group G0 contributes steps K0LAST.. only (first group of
  // half 1), group G1 steps ..KLAST; columns from C0
#pragma unroll
  for (int g = G0; g <= G1; ++g) {
    uint32_t s = __byte_perm(wq[(g >> 1) - wbase], 0u, (g & 1) ? 0x4342u : 0x4140u);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t p = s * 3u;
      const int c = C0 + 5 * (g - G0) + k - K0LAST;
      if (!(g == G0 && k < K0LAST) && !(g == G1 && k > KLAST)) col[c] = q1_trit2<T>(p);
      s = p & 0x00FF00FFu;
    }
  }
}
template <typename T>
__device__ __forceinline__ void decode_q1(const uint32_t (&wq)[7], int half, uint32_t (&col)[64]) {
  if (half == 0) q1_groups<T, 0, 12, 0, 3, 0>(wq, 0, col);     // cols 0..63
  else q1_groups<T, 12, 25, 4, 2, 0>(wq, 6, col);              // cols 64..127 (as 0..63)
}

}  // namespace umma

struct UmmaArgs {
  const uint8_t* w;   // T16 units, tile-major
  void* y;            // [batch][ldy]
  float* ws;          // split-K partials
  int* counters;      // per-(m, n) tile arrival counters (zero between launches)
  int64_t ldy;
  int rows, nb, batch;
  int m_tiles, n_tiles, ks;
  int uniform;        // every row has one scale for all its blocks
  int dbg;            // development probes: 1 = skip MMAs, 2 = skip decode/TMEM stores, 4 = CTA 0 clock
                      // trace into y (no output): per block, MMA warp [0] activations landed [1] A
                      // decoded [2] MMAs issued; decode warp 0 [3] A buffer free [4] TMEM stores done
  int map3d;          // activations described by the 3-D tensor map (one TMA request per block)
  int out_f32;        // TR_LINEAR_OUT_F32: y is float32
  int epi;            // TR_LINEAR_EPI_SWIGLU: rows are 16-row gate / up tile pairs; y[:, rows / 2] = silu(gate) * up
};

// SwiGLU store of one warp's 32 rows (a gate tile in lanes 0-15, its up tile in lanes 16-31) for
// activation rows n0.., with the roundings of the unfused gate|up store + tr_silu_mul
template <typename T, int NV>
__device__ __forceinline__ void store_swiglu(const UmmaArgs& a, const float (&v)[NV], int n0, int pair, int lane) {
  const int orow = pair * 16 + (lane & 15);
#pragma unroll
  for (int e = 0; e < NV; ++e) {
    const float g = Act<T>::to_float(Act<T>::from_float(v[e]));
    const float u = Act<T>::to_float(Act<T>::from_float(__shfl_xor_sync(0xffffffffu, v[e], 16)));
    const float sg = Act<T>::to_float(Act<T>::from_float(__fdividef(g, 1.0f + __expf(-g))));
    if (lane < 16 && n0 + e < a.batch) store_y<T>(a.y, (int64_t)(n0 + e) * a.ldy + orow, sg * u, 0);
  }
}

template <typename T, int N, int FMT>
struct UmmaCfg {
  static constexpr int UB = FMT == kFmtTq1 ? kQ1UnitBytes : kUnitBytes;   // bytes per 16x256 unit
  static constexpr int TBB = FMT == kFmtTq1 ? kQ1TileBlockBytes : kTileBlockBytes;
  // TMA requests cost ~100 SM cycles each whatever their size, so the weights move in
  // stages of KS blocks (8 requests of KS x 1056 B) and the activations in one 3-D box per block
#ifndef UMMA_N128_RB
#define UMMA_N128_RB 3
#endif
  // N = 128: three 64 KB activation stages and two weight stages (exactly 227 KB).  The
  // activation ring's turnaround (commit -> refill -> landed) bounds the block rate, so its
  // depth matters more than the weight ring's
#ifndef UMMA_KS_SMALL
#define UMMA_KS_SMALL 4
#endif
#ifndef UMMA_RW_SMALL
#define UMMA_RW_SMALL 4   // (N = 32 only: N = 16 has UMMA_RW16)
#endif
#ifndef UMMA_RB16
#define UMMA_RB16 4
#endif
  static constexpr int KS = N <= 32 ? UMMA_KS_SMALL : 2;     // 256-blocks per weight stage
  // weight stages: two at N = 64 / 128 (re-measured after the MMA issue work: N = 64 4096^2 b=128
  // 10.96 -> 10.58 us, 4096x11008 b=64 13.35 -> 13.12 against three).  N = 16 / 32 take four since
  // K5's interleaved decode (the weight ring underflowed every stage of KS blocks): N = 16 with four
  // 8 KB activation stages (stack b=8-16 -5%), N = 32 with three 16 KB ones (stack b=24-32 -1.9%)
#ifndef UMMA_RW_MID
#define UMMA_RW_MID 2
#endif
#ifndef UMMA_RB_MID
#define UMMA_RB_MID 5
#endif
#ifndef UMMA_RW16
#define UMMA_RW16 4
#endif
  static constexpr int RW = N <= 16 ? UMMA_RW16 : N <= 32 ? UMMA_RW_SMALL : (N == 128 && UMMA_N128_RB == 3) ? 2 : UMMA_RW_MID;
  // (N = 64: the spare shared memory goes to activation stages, +0.5-1.2% at b = 64; N = 16 / 32
  // measured best with four weight stages instead, above)
#ifndef UMMA_RB32
#define UMMA_RB32 3
#endif
  static constexpr int RB = N <= 16 ? UMMA_RB16 : N <= 32 ? UMMA_RB32 : N <= 64 ? UMMA_RB_MID : UMMA_N128_RB;   // activation stages (one block each)
  static constexpr int kStageWBytes = 8 * KS * UB;          // 128 rows x KS blocks
  static constexpr int kStageBBytes = N * 512;               // N rows x 256 K (4 swizzled 64-K atoms)
  static constexpr int kMaxA = 3;                            // TMEM A buffers (128 columns = one block each)
  static constexpr size_t kBOff = 1024;                      // 1024-aligned for the 128B swizzle
  static constexpr size_t kWOff = kBOff + (size_t)RB * kStageBBytes;
  static constexpr size_t kSmem = kWOff + (size_t)RW * kStageWBytes + 1024;   // + alignment slack
  static_assert(kSmem <= 227 * 1024, "K5 stages exceed the shared memory of one CTA");
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(r) : "r"(addr));
  return r;
}

// SPLIT: the product is split along K (a.ks > 1).  The unsplit instance carries no reduction code:
// its mere presence cost the unsplit product ~6% (11008x4096 b=16: 10.0 vs 9.4 us), through the
// register allocation of the decode and MMA loops
template <typename T, int N, int FMT, bool SPLIT, bool EPI>
__global__ void __launch_bounds__(umma::kThreads, 1)
    k_gemm_umma(const __grid_constant__ CUtensorMap tmx, const UmmaArgs a) {
  using namespace umma;
  using Cfg = UmmaCfg<T, N, FMT>;
  constexpr int UB = Cfg::UB;
  constexpr int KS = Cfg::KS, RW = Cfg::RW, RB = Cfg::RB;
  constexpr int kStageW = Cfg::kStageWBytes, kStageB = Cfg::kStageBBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_w = reinterpret_cast<uint64_t*>(smem);     // RW
  uint64_t* empty_w = full_w + RW;                           // RW
  uint64_t* full_b = empty_w + RW;                           // RB
  uint64_t* empty_b = full_b + RB;                           // RB
  uint64_t* a_full = empty_b + RB;                           // kMaxA
  uint64_t* a_empty = a_full + Cfg::kMaxA;                   // kMaxA
  uint64_t* d_full = a_empty + Cfg::kMaxA;                   // 2
  uint64_t* d_empty = d_full + 2;                            // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);
  uint8_t* sB = smem + Cfg::kBOff;
  uint8_t* sW = smem + Cfg::kWOff;

  // activation ring and TMEM A ring of the same depth (N <= 64: NA = kMaxA = 3 in both scale modes):
  // one commit per block releases both, and the producer waits on the A ring's barrier.  Applies to
  // N = 32 (three activation stages): stack b=32 0.869 -> 0.857 ms; at N = 16 it only recovers what
  // a third activation stage instead of four costs
  constexpr bool kMergeB = UMMA_MERGE && RB == Cfg::kMaxA && N <= 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x % a.m_tiles;
  const int nt = (blockIdx.x / a.m_tiles) % a.n_tiles;
  const int kslice = blockIdx.x / (a.m_tiles * a.n_tiles);
  const int kb0 = (int)((int64_t)kslice * a.nb / a.ks), kb1 = (int)((int64_t)(kslice + 1) * a.nb / a.ks);
  const int nblk = kb1 - kb0;
  const int nws = (nblk + KS - 1) / KS;   // weight stages
  const bool per_block = !a.uniform;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RW; ++s) {
      mbar_init(&full_w[s], 1);
      mbar_init(&empty_w[s], kWorkers);
    }
    for (int s = 0; s < RB; ++s) {
      mbar_init(&full_b[s], 1);
      mbar_init(&empty_b[s], 1);
    }
    for (int i = 0; i < Cfg::kMaxA; ++i) {
      mbar_init(&a_full[i], (kIlv && N <= UMMA_ILV_MAXN && !per_block) ? kWorkers / 2 : kWorkers);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], kWorkers);
    }
    mbar_fence_init();
  }
  if (warp == kWorkers + 1) {   // TMEM: A double buffer (2 x 128 cols) + D (2 x N cols)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: NA A buffers of 128 columns, then the accumulator(s): 2 x N (per-block, double
  // buffered) or N (uniform scale, one accumulator over all K)
  const int dcols = per_block ? 2 * N : N;
  const int NA = (512 - dcols) / 128 < Cfg::kMaxA ? (512 - dcols) / 128 : Cfg::kMaxA;
  const uint32_t tA = tmem, tD = tmem + NA * 128;
  if (tmem != 0u && threadIdx.x == 0) __trap();   // 512 columns: the whole TMEM, so address 0 (see MMA warp)
  griddep_launch_dependents();

  if (warp == kWorkers) {
    // ================= TMA producer (one thread) =================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmx) : "memory");
      const uint64_t pol = policy_evict_first();
      const uint8_t* wbase = a.w + ((int64_t)mt * 8 * a.nb + kb0) * UB;
      auto issue_w = [&](int si) {   // weight stage si: blocks [si KS, si KS + c) of the CTA's 8 tiles
        const int s = si % RW, c = min(KS, nblk - si * KS);
        mbar_expect_tx(&full_w[s], 8 * c * UB);
#pragma unroll 1
        for (int t = 0; t < 8; ++t)
          bulk_g2s(sW + s * kStageW + t * KS * UB, wbase + ((int64_t)t * a.nb + si * KS) * UB, c * UB, &full_w[s],
                   pol);
      };
      auto issue_b = [&](int i) {
        const int s = i % RB;
        mbar_expect_tx(&full_b[s], kStageB);
        if (a.map3d) {
          tma_load_3d(sB + s * kStageB, &tmx, 0, nt * N, (kb0 + i) * 4, &full_b[s]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            tma_load_2d(sB + s * kStageB + q * N * 128, &tmx, (kb0 + i) * kBlock + q * 64, nt * N, &full_b[s]);
        }
      };
      int nw_ = nws < RW ? nws : RW, nb_ = nblk < RB ? nblk : RB;
      for (int si = 0; si < nw_; ++si) issue_w(si);   // weights do not depend on the previous kernel
      griddep_wait();
      for (int i = 0; i < nb_; ++i) issue_b(i);
      while (nw_ < nws || nb_ < nblk) {                // refill whichever ring is needed first
        if (nw_ < nws && (nw_ * KS <= nb_ || nb_ >= nblk)) {
          mbar_wait(&empty_w[nw_ % RW], ((nw_ / RW) & 1) ^ 1);
          issue_w(nw_++);
        } else {
          if (kMergeB) mbar_wait(&a_empty[nb_ % RB], ((nb_ / RB) & 1) ^ 1);   // (same ring: one commit)
          else mbar_wait(&empty_b[nb_ % RB], ((nb_ / RB) & 1) ^ 1);
          issue_b(nb_++);
        }
      }
    }
  } else if (warp == kWorkers + 1) {
    // ================= MMA issuer (one thread) =================
    constexpr uint32_t kFmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
    constexpr uint32_t idesc = (1u << 4) | (kFmt << 7) | (kFmt << 10) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(kRowsPerCta >> 4) << 24);
    // shared-window address of the activation stages from the (uniform) dynamic-smem base, so the
    // MMA descriptors are computed in uniform registers rather than moved there once per MMA
    const uint32_t sB32 = ((smem_u32(smem_raw) + 1023u) & ~1023u) + (uint32_t)Cfg::kBOff;
    {   // the whole warp runs the loop; each MMA / commit is issued by one elected lane
      int s = 0, bph = 0, ab = 0, aph = 0;
      for (int i = 0; i < nblk; ++i) {
        const int db = i & 1;
        mbar_wait(&full_b[s], bph);                  // activations landed
        if (kTrace && (a.dbg & 4) && blockIdx.x == 0 && lane == 0 && i < 64)
          reinterpret_cast<long long*>(a.y)[i * 8 + 0] = clock64();
        mbar_wait(&a_full[ab], aph);                 // trits decoded into TMEM
        if (kTrace && (a.dbg & 4) && blockIdx.x == 0 && lane == 0 && i < 64)
          reinterpret_cast<long long*>(a.y)[i * 8 + 1] = clock64();
        if (per_block) mbar_wait(&d_empty[db], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        // (the CTA allocates all 512 TMEM columns, so the allocation starts at address 0: the MMA
        // addresses are compile-time / loop-uniform values in uniform registers, not a shared-memory
        // load moved into uniform registers before every MMA -- checked once below)
        const uint32_t d = per_block ? (uint32_t)(NA * 128 + db * N) : (uint32_t)(NA * 128);
        // the block's 16 MMAs (K = 256) from one asm block, one elect, descriptors built in the
        // uniform datapath (measured: b=16 -7%, b=64 -6%, b=128 -10% per layer against one MMA per
        // call with descriptors moved in from ordinary registers)
        if (!(a.dbg & 1))
          mma_block16<N>(d, (uint32_t)(ab * 128), sB32 + s * kStageB, idesc, (!per_block && i > 0) ? 1 : 0);
        if (kTrace && (a.dbg & 4) && blockIdx.x == 0 && lane == 0 && i < 64)
          reinterpret_cast<long long*>(a.y)[i * 8 + 2] = clock64();
        if (!kMergeB) mma_commit(&empty_b[s]);       // activation stage reusable once these MMAs finish
        mma_commit(&a_empty[ab]);                    // TMEM A buffer reusable
        if (per_block || i == nblk - 1) mma_commit(&d_full[per_block ? db : 0]);
        if (++s == RB) {   // (ring positions and phases advance incrementally)
          s = 0;
          bph ^= 1;
        }
        if (++ab == NA) {
          ab = 0;
          aph ^= 1;
        }
        if (kTrace && (a.dbg & 4) && blockIdx.x == 0 && lane == 0 && i < 64)
          reinterpret_cast<long long*>(a.y)[i * 8 + 5] = clock64();
      }
    }
  } else {
    // ================= decode + epilogue warps =================
    const int quad = warp & 3, half_k = warp >> 2;     // TMEM lanes 32 quad..; K chunks 2 half_k, +1
    const int r = quad * 32 + lane;                    // row within the CTA tile
    const int tl = r >> 4, rt = r & 15;                // T16 tile, row in tile
    const int hrow = rt >> 3, g = rt & 7;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    constexpr int NH = N / 2;                          // epilogue columns per thread
    float acc[NH];
#pragma unroll
    for (int i = 0; i < NH; ++i) acc[i] = 0.0f;
    float s_prev = 0.0f, s_first = 0.0f;
    const uint32_t sW32 = smem_u32(sW) + tl * KS * UB;

    auto epilogue_block = [&](int i, float s) {        // acc += s * D_i (this thread's half of N)
      const int ab = i & 1;
      mbar_wait(&d_full[ab], (i >> 1) & 1);
      tc_fence_after();
      // all of this thread's NH columns in flight at once (x32 / x16 / x8 loads), one wait
      constexpr int NC = NH >= 32 ? 32 : NH;
      uint32_t v[NH / NC][NC];
#pragma unroll
      for (int c = 0; c < NH / NC; ++c) tmem_ld_cols<NC>(tD + lane_off + ab * N + half_k * NH + c * NC, v[c]);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < NH / NC; ++c)
#pragma unroll
        for (int e = 0; e < NC; ++e) acc[c * NC + e] = fmaf(s, __uint_as_float(v[c][e]), acc[c * NC + e]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d_empty[ab]);
    };

    auto finish_block = [&](int i, float s_cur, int ab) {
      tmem_wait_st();
      if (kTrace && (a.dbg & 4) && blockIdx.x == 0 && lane == 0 && i < 64 && (warp == 0 || warp == 1 || warp == 6))
        reinterpret_cast<long long*>(a.y)[i * 8 + (warp == 0 ? 4 : warp == 1 ? 6 : 7)] = clock64();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[ab]);
      if (i == 0) s_first = s_cur;
      if (per_block && i > 0) epilogue_block(i - 1, s_prev);
      s_prev = s_cur;
    };
    if (kIlv && N <= UMMA_ILV_MAXN && !per_block) {
      // uniform scale (no per-block epilogue): the two warp groups decode alternate 256-blocks, each
      // a whole block of its 32 rows, so one group's per-block waits (weights, A buffer, TMEM store
      // drain) overlap the other group's decode.  Every warp still arrives once per weight stage
      // (KS >= 2: a stage holds blocks of both parities, except a one-block last stage, which is
      // never refilled); A buffers i % kMaxA (NA = kMaxA in this mode).  Measured (umma_b16.py):
      // b=16-32 2-3% faster per layer; at N = 64 / 128 1-4% slower (MMA-paced there), so N <= 32
      constexpr int NAu = Cfg::kMaxA;
      bool have_s = false;
      for (int i = half_k; i < nblk; i += 2) {
        const int j = i % KS, si = i / KS, s = si % RW;
        if (j < 2) mbar_wait(&full_w[s], (si / RW) & 1);
        const uint32_t unit = sW32 + s * kStageW + j * UB;
        const uint32_t sv = ld_shared_u32(unit + Cfg::TBB + g * 4);
        uint4 wv[4];
        uint32_t wq[2][7];
        if constexpr (FMT == kFmtTq1) {
#pragma unroll
          for (int hk = 0; hk < 2; ++hk)
#pragma unroll
            for (int m = 0; m < 7; ++m) wq[hk][m] = ld_shared_u32(unit + rt * kQ1RowBytes + (hk * 6 + m) * 4);
        } else {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) wv[cc] = ld_shared_v4(unit + t16_word(hrow, cc, g) * 16);
        }
        if (!have_s) {
          s_first = __half2float(hrow ? __high2half(*reinterpret_cast<const __half2*>(&sv))
                                      : __low2half(*reinterpret_cast<const __half2*>(&sv)));
          have_s = true;
        }
        if (j + 2 >= KS || i + 2 >= nblk) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_w[s]);
        }
        const int ab = i % NAu;
        mbar_wait(&a_empty[ab], ((i / NAu) & 1) ^ 1);
        tc_fence_after();
        if (!(a.dbg & 2)) {
          if constexpr (FMT == kFmtTq1) {
#pragma unroll
            for (int hk = 0; hk < 2; ++hk) {
              uint32_t col[64];
              decode_q1<T>(wq[hk], hk, col);
              tmem_st32(tA + lane_off + ab * 128 + hk * 64, *reinterpret_cast<const uint32_t(*)[32]>(col));
              tmem_st32(tA + lane_off + ab * 128 + hk * 64 + 32, *reinterpret_cast<const uint32_t(*)[32]>(col + 32));
            }
          } else {
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              const uint32_t W[4] = {wv[cc].x, wv[cc].y, wv[cc].z, wv[cc].w};
              uint32_t col[32];
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                const uint32_t w8 = W[w] >> 8;
#pragma unroll
                for (int hb = 0; hb < 2; ++hb)
#pragma unroll
                  for (int jj = 0; jj < 4; ++jj)
                    col[16 * (w >> 1) + 8 * hb + 2 * jj + (w & 1)] = Dec<T>::trit2(W[w], w8, hb, jj);
              }
              tmem_st32(tA + lane_off + ab * 128 + cc * 32, col);
            }
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[ab]);
      }
      if (!have_s && nblk > 0) {   // one block, taken by the other group: its scale (single stage)
        mbar_wait(&full_w[0], 0);
        const uint32_t sv = ld_shared_u32(sW32 + Cfg::TBB + g * 4);
        s_first = __half2float(hrow ? __high2half(*reinterpret_cast<const __half2*>(&sv))
                                    : __low2half(*reinterpret_cast<const __half2*>(&sv)));
      }
    } else {   // per block: weights to registers, wait for the A buffer, decode 32 columns at a time into TMEM
      // (ring positions and phases advance incrementally: the divisions by KS, RW and NA were a
      // tenth of the decode warps' instructions at N = 16)
      int j = 0, s = 0, wph = 0, ab = 0, aph = 1;
      for (int i = 0; i < nblk; ++i) {
        if (j == 0) mbar_wait(&full_w[s], wph);
        const uint32_t unit = sW32 + s * kStageW + j * UB;
        uint4 wv[2];
        uint32_t wq[7];
        if constexpr (FMT == kFmtTq1) {
#pragma unroll
          for (int m = 0; m < 7; ++m) wq[m] = ld_shared_u32(unit + rt * kQ1RowBytes + (half_k * 6 + m) * 4);
        } else {
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) wv[cc] = ld_shared_v4(unit + t16_word(hrow, 2 * half_k + cc, g) * 16);
        }
        const uint32_t sv = ld_shared_u32(unit + Cfg::TBB + g * 4);
        const float s_cur = __half2float(hrow ? __high2half(*reinterpret_cast<const __half2*>(&sv))
                                              : __low2half(*reinterpret_cast<const __half2*>(&sv)));
        if (j == KS - 1 || i == nblk - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_w[s]);
        }
        mbar_wait(&a_empty[ab], aph);
        if (kTrace && (a.dbg & 4) && blockIdx.x == 0 && threadIdx.x == 0 && i < 64)
          reinterpret_cast<long long*>(a.y)[i * 8 + 3] = clock64();
        tc_fence_after();
        if constexpr (FMT == kFmtTq1) {
          if (!(a.dbg & 2)) {
            uint32_t col[64];
            decode_q1<T>(wq, half_k, col);
            tmem_st32(tA + lane_off + ab * 128 + half_k * 64, *reinterpret_cast<const uint32_t(*)[32]>(col));
            tmem_st32(tA + lane_off + ab * 128 + half_k * 64 + 32, *reinterpret_cast<const uint32_t(*)[32]>(col + 32));
          }
        } else
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          if (a.dbg & 2) break;
          const uint32_t W[4] = {wv[cc].x, wv[cc].y, wv[cc].z, wv[cc].w};
          uint32_t col[32];
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const uint32_t w8 = W[w] >> 8;
#pragma unroll
            for (int hb = 0; hb < 2; ++hb)
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
                col[16 * (w >> 1) + 8 * hb + 2 * jj + (w & 1)] = Dec<T>::trit2(W[w], w8, hb, jj);
          }
          tmem_st32(tA + lane_off + ab * 128 + (2 * half_k + cc) * 32, col);
        }
        finish_block(i, s_cur, ab);
        if (++j == KS) {
          j = 0;
          if (++s == RW) {
            s = 0;
            wph ^= 1;
          }
        }
        if (++ab == NA) {
          ab = 0;
          aph ^= 1;
        }
      }
    }
    if (nblk > 0) {
      if (per_block) epilogue_block(nblk - 1, s_prev);
      else epilogue_block(0, s_first);   // the single accumulator (committed after the last block)
    }
    griddep_wait();
    // ---- store: whole K in this CTA -> y; else partials + last-CTA reduction (fixed slice order)
    const int row = mt * kRowsPerCta + r;
    const int n0 = nt * N + half_k * NH;
    // (SwiGLU: rows % 32 == 0, so a warp's 32 rows are all in range or all out, and the gate / up
    // shuffle runs warp-wide)
    const int pair = mt * 4 + quad;
    if (!SPLIT || (a.dbg & 8)) {   // (dev probe 8: split-K slices store unreduced -- timing only)
      if (row < a.rows && !(kTrace && (a.dbg & 4))) {
        if constexpr (EPI) {
          store_swiglu<T, NH>(a, acc, n0, pair, lane);
        } else {
#pragma unroll
          for (int e = 0; e < NH; ++e)
            if (n0 + e < a.batch) store_y<T>(a.y, (int64_t)(n0 + e) * a.ldy + row, acc[e], a.out_f32);
        }
      }
    } else if constexpr (SPLIT) {
      const int tile_mn = nt * a.m_tiles + mt;
      float* part = a.ws + ((int64_t)tile_mn * a.ks + kslice) * (kRowsPerCta * N);
#pragma unroll
      for (int e = 0; e < NH; ++e) __stcg(part + (half_k * NH + e) * kRowsPerCta + r, acc[e]);
      __threadfence();
      asm volatile("bar.sync 1, %0;\n" ::"n"(kWorkers * 32) : "memory");   // all workers stored
      if (threadIdx.x == 0) *flag = atomicAdd(a.counters + tile_mn, 1) == a.ks - 1;
      asm volatile("bar.sync 1, %0;\n" ::"n"(kWorkers * 32) : "memory");
      if (*flag) {   // the last CTA of this tile sums the ks partials in slice order
        __threadfence();
        const float* base = a.ws + (int64_t)tile_mn * a.ks * (kRowsPerCta * N);
        // up to 32 independent loads in flight per slice (the sum is latency-bound: one L2 round
        // trip per slice and chunk)
        constexpr int EC = NH < 32 ? NH : 32;
        if (row < a.rows && !(kTrace && (a.dbg & 4)))
#pragma unroll
          for (int e0 = 0; e0 < NH; e0 += EC) {
            float v[EC];
#pragma unroll
            for (int e = 0; e < EC; ++e) v[e] = 0.0f;
            // QB slices' loads in flight before any of them is added (in program order the adds
            // of one slice would hold back the next slice's loads: one L2 round trip per slice)
            constexpr int QB = 64 / EC;
            for (int q0 = 0; q0 < a.ks; q0 += QB) {
              float u[QB][EC];   // (this CTA's own slice too: taking it from registers measured slower)
#pragma unroll
              for (int qq = 0; qq < QB; ++qq) {
                const float* src =
                    base + (int64_t)(q0 + qq) * kRowsPerCta * N + (half_k * NH + e0) * kRowsPerCta + r;
#pragma unroll
                for (int e = 0; e < EC; ++e) u[qq][e] = q0 + qq < a.ks ? __ldcg(src + e * kRowsPerCta) : 0.0f;
              }
#pragma unroll
              for (int qq = 0; qq < QB; ++qq)   // slice order (the zeros past ks leave the sum unchanged)
#pragma unroll
                for (int e = 0; e < EC; ++e) v[e] += u[qq][e];
            }
            if constexpr (EPI) {
              store_swiglu<T, EC>(a, v, n0 + e0, pair, lane);
            } else {
#pragma unroll
              for (int e = 0; e < EC; ++e)
                if (n0 + e0 + e < a.batch) store_y<T>(a.y, (int64_t)(n0 + e0 + e) * a.ldy + row, v[e], a.out_f32);
            }
          }
        if (threadIdx.x == 0) a.counters[tile_mn] = 0;   // self-reset
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kWorkers + 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ------------------------------------------------------------------------------------ host

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

constexpr size_t kUmmaCounterBytes = 256 * 1024;   // per-(m, n) tile counters (the workspace's fixed counter region)

struct UmmaPlan {
  int n, n_tiles, m_tiles, ks;
  size_t ws_bytes;
};

static UmmaPlan plan_umma(int batch, int rows, int cols, int ks_force, int sms) {
  UmmaPlan p;
  p.n = batch <= 16 ? 16 : batch <= 32 ? 32 : batch <= 64 ? 64 : 128;
  p.m_tiles = (int)(rows_padded(rows) / 128);
  // few row tiles, wide batch, short K: two half-width column tiles per row tile and half the K
  // split -- the same MMA work per CTA, half the slices (each half the bytes) to sum, which
  // dominates when each CTA walks only a few blocks (4096^2: b=128 14.1 -> 11.0 us, b=64 9.5 ->
  // 9.0; with 43 blocks of K the narrower MMAs cost more than the sum saves: 4096x11008 b=64
  // 13.4 -> 16.4)
  if (ceil_div(cols, kBlock) <= 16 && 2 * p.m_tiles <= sms && p.n >= 64) p.n /= 2;
  p.n_tiles = (int)ceil_div(batch, p.n);
  const int nb = (int)ceil_div(cols, kBlock);
  const int base = p.m_tiles * p.n_tiles;
  int ks = ks_force > 0 ? ks_force : (base >= sms ? 1 : sms / base);
  if (ks > nb / 2) ks = nb / 2 > 0 ? nb / 2 : 1;
  if (ks > 16) ks = 16;
  if (ks < 1) ks = 1;
  p.ks = ks;
  p.ws_bytes = ks > 1 ? (size_t)base * ks * 128 * p.n * 4 : 0;
  return p;
}

// 256-blocks of K each K5 CTA walks for this product (its split-K share): the dispatcher's
// measure of how well the tensor-core GEMM spreads a shape over the SMs
int umma_blocks_per_cta(int batch, int rows, int cols) {
  const UmmaPlan p = plan_umma(batch, rows, cols, 0, sm_count());
  return (int)ceil_div(ceil_div(cols, kBlock), p.ks);
}

size_t umma_workspace_bytes(int batch, int rows, int cols) {
  size_t ws = 0;
  for (int ks = 0; ks <= 16; ++ks) {
    UmmaPlan p = plan_umma(batch, rows, cols, ks, sm_count());
    if (p.ws_bytes > ws) ws = p.ws_bytes;
  }
  return kUmmaCounterBytes + ws;
}

template <typename T, int N, int FMT>
static int launch_umma(const CUtensorMap& map, const UmmaArgs& a, int grid, int pdl, cudaStream_t st) {
  // (SwiGLU store: its own instances, TQ2 only -- a runtime branch in the shared store code cost
  // b=128 3.8% and b=64 2% through the register allocation, as the split-K sum once did)
  auto kern = a.ks > 1 ? k_gemm_umma<T, N, FMT, true, false> : k_gemm_umma<T, N, FMT, false, false>;
  if constexpr (FMT == kFmtTq2)
    if (a.epi) kern = a.ks > 1 ? k_gemm_umma<T, N, FMT, true, true> : k_gemm_umma<T, N, FMT, false, true>;
  const int inst = (a.ks > 1) + 2 * (a.epi != 0);
  static int configured_dev[4] = {-1, -1, -1, -1};
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev[inst] != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)UmmaCfg<T, N, FMT>::kSmem);
    configured_dev[inst] = dev;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(umma::kThreads, 1, 1);
  cfg.dynamicSmemBytes = UmmaCfg<T, N, FMT>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  int na = 0;
  if (pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, map, a);
  if (e != cudaSuccess) {
    set_error("tr_linear(umma): launch failed: %s (grid %d)", cudaGetErrorString(e), grid);
    return -1;
  }
  return 0;
}

int gemm_umma(int fmt, int act, const void* w, const void* x, void* y, int64_t ldx, int64_t ldy, int batch, int rows,
              int cols, int ks, int uniform, void* workspace, size_t ws_bytes, int pdl, cudaStream_t st, int dbg,
              int out_f32, int epi) {
  UmmaPlan p = plan_umma(batch, rows, cols, ks, sm_count());
  if ((ldx % 8) != 0 || ((uintptr_t)x & 15) != 0) {
    set_error("tr_linear(umma): activations need 16-byte aligned rows (ldx %% 8 == 0)");
    return -1;
  }
  if ((size_t)p.m_tiles * p.n_tiles * 4 > kUmmaCounterBytes || workspace == nullptr ||
      ws_bytes < kUmmaCounterBytes + p.ws_bytes) {
    set_error("tr_linear(umma): workspace too small (%zu < %zu)", ws_bytes, kUmmaCounterBytes + p.ws_bytes);
    return -1;
  }
  EncodeTiledFn enc = encode_fn();
  if (!enc) {
    set_error("tr_linear(umma): cuTensorMapEncodeTiled unavailable");
    return -1;
  }
  CUtensorMap map;
  const CUtensorMapDataType dt = act == kActBf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  int map3d = 0;
  CUresult cr = CUDA_ERROR_INVALID_VALUE;
  if (cols % kBlock == 0) {   // x as [cols/64][batch][64]: one request loads a whole 256-block
    const cuuint64_t dims[3] = {64, (cuuint64_t)batch, (cuuint64_t)(cols / 64)};
    const cuuint64_t strides[2] = {(cuuint64_t)ldx * 2, 128};
    const cuuint32_t box[3] = {64, (cuuint32_t)p.n, 4};
    const cuuint32_t estr[3] = {1, 1, 1};
    cr = enc(&map, dt, 3, const_cast<void*>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    map3d = cr == CUDA_SUCCESS;
  }
  if (!map3d) {
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)batch};
    const cuuint64_t strides[1] = {(cuuint64_t)ldx * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)p.n};
    const cuuint32_t estr[2] = {1, 1};
    cr = enc(&map, dt, 2, const_cast<void*>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (cr != CUDA_SUCCESS) {
    set_error("tr_linear(umma): cuTensorMapEncodeTiled failed (%d)", (int)cr);
    return -1;
  }
  UmmaArgs a;
  a.w = (const uint8_t*)w;
  a.y = y;
  a.counters = (int*)workspace;
  a.ws = (float*)((uint8_t*)workspace + kUmmaCounterBytes);
  a.ldy = ldy;
  a.rows = rows;
  a.nb = (int)ceil_div(cols, kBlock);
  a.batch = batch;
  a.m_tiles = p.m_tiles;
  a.n_tiles = p.n_tiles;
  a.ks = p.ks;
  a.uniform = uniform;
  a.dbg = dbg;
  a.map3d = map3d;
  a.out_f32 = out_f32;
  a.epi = epi;
  if (epi && (rows % 32 != 0 || out_f32 || fmt != kFmtTq2)) {
    set_error("tr_linear(umma, swiglu epilogue): rows (%d) must be whole 32-row gate/up pairs, fp16/bf16 out", rows);
    return -1;
  }
  const int grid = p.m_tiles * p.n_tiles * p.ks;
  const bool bf = act == kActBf16;
#define TR_UMMA_CASE(NN)                                                                              \
  case NN:                                                                                            \
    if (fmt == kFmtTq1)                                                                               \
      return bf ? launch_umma<__nv_bfloat16, NN, kFmtTq1>(map, a, grid, pdl, st)                      \
                : launch_umma<__half, NN, kFmtTq1>(map, a, grid, pdl, st);                            \
    return bf ? launch_umma<__nv_bfloat16, NN, kFmtTq2>(map, a, grid, pdl, st)                        \
              : launch_umma<__half, NN, kFmtTq2>(map, a, grid, pdl, st);
  switch (p.n) {
    TR_UMMA_CASE(16)
    TR_UMMA_CASE(32)
    TR_UMMA_CASE(64)
    default:
    TR_UMMA_CASE(128)
  }
#undef TR_UMMA_CASE
}

}  // namespace tr
