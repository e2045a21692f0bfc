// Shared definitions for the B200 (sm_100a) TriRun kernels.
//
// Formats follow the reference package `tritpack` (blocks.py:34-86): a block is
// 256 consecutive K-elements of one row; TQ2 = 64 payload bytes (4 digits per
// byte, element 4t+j at bits 2j), TQ1 = 52 payload bytes (5 digits per byte,
// base-3, MSB first); one binary16 scale per (row, block).  Digits are
// d = trit + 1 in {0, 1, 2}.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "tritrun.h"

namespace tr {

constexpr int kBlock = 256;         // BLOCK_ELEMENTS (blocks.py:34)
constexpr int kTq2Payload = 64;     // DType.TQ2.payload_bytes (blocks.py:63-70)
constexpr int kTq1Payload = 52;     // DType.TQ1.payload_bytes
constexpr int kFmtTq2 = 2;          // DType.TQ2 (blocks.py:49-52)
constexpr int kFmtTq1 = 3;          // DType.TQ1
constexpr int kActF16 = 1;
constexpr int kActBf16 = 2;
constexpr int kActF32 = 3;

// ---- T16 device layout -----------------
// Rows are padded to a multiple of 128 (zero trits, zero scales).  The matrix is
// cut into 16-row tiles t and 256-column blocks b; unit (t, b) is 1056 contiguous
// bytes at offset (t * nb + b) * 1056 (tile-major, so a tile's K range is one
// contiguous run that a single TMA bulk copy can fetch):
//   bytes [0, 1024): 64 16-byte words; word u = half*32 + c*8 + (g ^ 2c) is chunk c
//     (block columns 64c..64c+63) of row 16t + 8*half + g (the XOR puts the 8 words an
//     MMA quarter-warp reads -- rows g, g^1 of all 4 chunks -- in 8 distinct bank groups),
//     encoded so that
//     32-bit word w (0..3), bits 16h + 8hb + 2j (+1), hold the digit of chunk
//     column 32*(w>>1) + 16hb + 4j + 2*(w&1) + h;
//   bytes [1024, 1056): 8 half2 scale pairs (s[16t+g], s[16t+8+g]).
constexpr int kRowPad = 128;
constexpr int kTileBlockBytes = 1024;
constexpr int kTileScaleBytes = 32;
constexpr int kUnitBytes = kTileBlockBytes + kTileScaleBytes;   // 1056
__host__ __device__ inline int t16_word(int half, int c, int g) { return half * 32 + c * 8 + (g ^ (2 * c)); }

// ---- T16-Q1 device layout for TQ1 (1.6 bit, 5 trits per byte) -------------------
// Same tiling (16-row tiles x 256-column blocks, tile-major units, rows padded to 128),
// unit = 16 rows x 52 payload bytes + the same 32 bytes of half2 scale pairs.  Row r of
// a unit (bytes 52 r ..) holds 26 pair-groups: group g covers columns 10g .. 10g+9 as
// byte A_g = base-3 code of the even columns (10g, +2, +4, +6, +8) and byte B_g = code
// of the odd ones (10g+1, .. +9), MSB first, codes canonical (codec.py:180-200);
// columns >= 256 (group 25's last two steps) are pad digits 1.  Placing A_g | B_g << 16
// in one register, each Algorithm-1 step (p = 3s, digit = p >> 8, s = p & 0xFF) on both
// 16-bit lanes at once yields the half2 of columns (10g + 2k, 10g + 2k + 1): natural-order
// K pairs for the tensor core.  Same 54 B per 256 weights as the reference TQ1 block.
constexpr int kQ1RowBytes = 52;
constexpr int kQ1TileBlockBytes = 16 * kQ1RowBytes;              // 832
constexpr int kQ1UnitBytes = kQ1TileBlockBytes + kTileScaleBytes;   // 864

__host__ __device__ inline int unit_bytes(int fmt) { return fmt == 3 ? kQ1UnitBytes : kUnitBytes; }
__host__ __device__ inline int tile_block_bytes(int fmt) { return fmt == 3 ? kQ1TileBlockBytes : kTileBlockBytes; }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t rows_padded(int64_t rows) { return ceil_div(rows, kRowPad) * kRowPad; }

// ---- PTX helpers --------------------------------------------------------------
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t magic) {
  uint32_t r;
  // (a & mask) | magic  -> immLut = (0xF0 & 0xCC) | 0xAA = 0xEA
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(a), "r"(mask), "r"(magic));
  return r;
}

__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ldg_nc_u32(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];\n" : "=r"(r) : "l"(p));
  return r;
}

// ---- mbarrier / bulk-copy (TMA) PTX ----------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// global -> shared bulk copy (cp.async.bulk, the TMA engine's 1-D mode); completes tx bytes on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_nohint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ld_shared_v4u(uint32_t addr) {   // 16 B from a shared-window address
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  return *reinterpret_cast<const uint4*>(p);
}

int sm_count();   // multiprocessor count of the current device (cached)

// ---- activation type traits ----------------------------------------------------
template <typename T> struct Act;
template <> struct Act<__half> {
  static constexpr int kId = kActF16;
  __device__ static __half from_float(float v) { return __float2half_rn(v); }
  __device__ static float to_float(__half v) { return __half2float(v); }
};
template <> struct Act<__nv_bfloat16> {
  static constexpr int kId = kActBf16;
  __device__ static __nv_bfloat16 from_float(float v) { return __float2bfloat16_rn(v); }
  __device__ static float to_float(__nv_bfloat16 v) { return __bfloat162float(v); }
};

// output element i of y: the activation type (rounded once, RNE) or, with TR_LINEAR_OUT_F32,
// the fp32 accumulator itself (row-parallel partials that an all-reduce sums)
template <typename T>
__device__ __forceinline__ void store_y(void* y, int64_t i, float v, int f32) {
  if (f32)
    reinterpret_cast<float*>(y)[i] = v;
  else
    reinterpret_cast<T*>(y)[i] = Act<T>::from_float(v);
}

}  // namespace tr

// ---- error plumbing for the C-ABI ---------------------------------------------------
namespace tr {
void set_error(const char* fmt, ...);
int check_launch(const char* what);
}  // namespace tr

#define TR_REQUIRE(cond, ...)            \
  do {                                   \
    if (!(cond)) {                       \
      ::tr::set_error(__VA_ARGS__);      \
      return -1;                         \
    }                                    \
  } while (0)
