// K3: decode-side ternary GEMV / skinny GEMM (batch 1..32), TQ2 weights.
//
// Semantics (reference linear.py:1-13, _kernels.pyx:136-168; paper App. F):
//   y[n, r] = sum_b s[r, b] * (sum_{k in block b} trit[r, k] * x[n, k])
// fp16/bf16 activations; each 256-block's inner sum is accumulated in fp32 and
// scaled by the fp32 value of its binary16 scale; output rounded once (RNE).
//
// B200 design:
//  * persistent stream-K: the n_tiles x nb tile-blocks (16 rows x 256 cols,
//    1 KB + 32 B scales in the T16 layout) of each K-slice are split into equal
//    contiguous ranges, one per warp -- every SM gets the same bytes, no wave
//    quantization, any matrix shape;
//  * each warp prefetches its own tile-blocks with cp.async.bulk (TMA bulk
//    copies, complete_tx on an mbarrier) into a private NS-deep shared-memory
//    ring: deep memory-level parallelism without holding data in registers;
//    the first NS copies are issued before griddepcontrol.wait, so a
//    PDL-chained layer streams its weights while the previous layer finishes;
//  * decode: one AND per half2 (fp16 subnormal trick) feeding mma.sync.m16n8k16
//    A fragments directly, 4 field-class accumulators, per-block correction
//    C(x) staged with x (see Frag);
//  * tiles split between warps / K-slices are reduced through a small fp32
//    workspace with a per-tile arrival counter; the last arriver sums the
//    segments in a fixed order (deterministic, self-resetting counters).
#include "common.cuh"

namespace tr {

constexpr int kXChunkBytes = 144;               // 64 halves + 16 B pad (bank spread)
constexpr int kXBlockBytes = 4 * kXChunkBytes;  // one 256-block of one activation row
constexpr int kOpUnits = 4;   // units (1056 B) per TMA bulk copy

__host__ __device__ inline int x_row_stride(int kb) {
  int r = kb * kXBlockBytes;
  return (r % 128 == 64) ? r : r + 64;   // rows g, g+1 land in opposite bank halves
}

// ---- mbarrier / bulk-copy PTX ------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// Field decode.  A word holds 8 bit-fields per 16-bit half: field (hb, j) at
// bits 8hb + 2j.  One AND/LOP3 per half2 turns a field into a value linear in
// the digit d, A = base + m_j * d, where m_j depends on the field class j =
// (col >> 2) & 3 of the column.  The staged activations are pre-scaled per
// column, x' = x * f_j with f_j = F / m_j (exact power-of-two scaling), so every
// mma of a unit accumulates into ONE fp32 accumulator P = base * sum(x') +
// F * sum(d * x), and per 256-block
//     sum_k (d_k - 1) x_k  =  P / F - C,   C = sum_k x_k (1 + base * f_k / F)
// with C staged once per CTA next to x.
template <typename T> struct Frag;
template <> struct Frag<__half> {
  // fp16: exponent left zero -> subnormal half d * 4^j * 2^-24 (no offset, base 0);
  // F = 2^-22 so f_j = 4^(1-j) in {4, 1, 1/4, 1/16} (|x| <= 16376 stays finite).
  __host__ __device__ static constexpr float kFactor(int j) {
    return j == 0 ? 4.0f : j == 1 ? 1.0f : j == 2 ? 0.25f : 0.0625f;
  }
  static constexpr float kInvF = 4194304.0f;   // 2^22
  static constexpr float kBase = 0.0f;
  __device__ static uint32_t field(uint32_t w, uint32_t w8, int hb, int j) {
    return (hb ? w8 : w) & (0x00030003u << (2 * j));
  }
  __device__ static uint32_t scale2(uint32_t v, float f) {
    __half2 r = __hmul2(*reinterpret_cast<const __half2*>(&v), __float2half2_rn(f));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  __device__ static void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
};
template <> struct Frag<__nv_bfloat16> {
  // bf16 (7 mantissa bits): magic exponent 0x4300 -> A = 128 + m_j d with
  // m_j = 4^j for j < 3 (bits 0..5) and m_3 = 1 (bits 6..7 shifted down);
  // F = 1 so f_j = 1/m_j (exact, no underflow in bf16's exponent range).
  __host__ __device__ static constexpr float kFactor(int j) {
    return j == 0 ? 1.0f : j == 1 ? 0.25f : j == 2 ? 0.0625f : 1.0f;
  }
  static constexpr float kInvF = 1.0f;
  static constexpr float kBase = 128.0f;
  __device__ static uint32_t field(uint32_t w, uint32_t w8, int hb, int j) {
    if (j < 3) return ((hb ? w8 : w) & (0x00030003u << (2 * j))) | 0x43004300u;
    return ((w >> (hb ? 14 : 6)) & 0x00030003u) | 0x43004300u;
  }
  __device__ static uint32_t scale2(uint32_t v, float f) {
    __nv_bfloat162 r = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&v), __float2bfloat162_rn(f));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  __device__ static void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
};

template <typename T>
__device__ __forceinline__ float sum4(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ float sum4<__half>(uint32_t a, uint32_t b) {
  const float2 fa = __half22float2(*reinterpret_cast<const __half2*>(&a));
  const float2 fb = __half22float2(*reinterpret_cast<const __half2*>(&b));
  return (fa.x + fa.y) + (fb.x + fb.y);
}
template <>
__device__ __forceinline__ float sum4<__nv_bfloat16>(uint32_t a, uint32_t b) {
  const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a));
  const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b));
  return (fa.x + fa.y) + (fb.x + fb.y);
}

struct GemvArgs {
  const uint8_t* w;      // T16 units (1056 B: 16x256 tile-block + scale pairs), tile-major
  const void* x;         // [batch][ldx]
  void* y;               // [batch][ldy]
  float* ws;             // split-tile partial segments
  int* counters;         // per-tile arrival counters (zero between launches)
  int64_t ldx, ldy;
  int rows, cols, nb, n_tiles, batch;
  int ks;                // K slices
  int cps;               // CTAs per K slice
  int segs_per_slice;    // workspace segment slots per tile and slice
  int x_vec;
  int xrs;               // staged activation row stride (bytes)
  int dbg;               // diagnostics: bit0 skip math, bit1 skip x loads
};

template <int CW>
struct Split {
  // warp wi (0 .. cps*CW-1) of a slice with `units` tile-blocks owns [u0(wi), u0(wi+1))
  __device__ static int u0(int wi, int units, int W) { return (int)((int64_t)wi * units / W); }
  __device__ static int owner(int u, int units, int W) { return (int)(((int64_t)(u + 1) * W - 1) / units); }
};

template <typename T, int NT, int CW, int NOPS>
__global__ void __launch_bounds__(CW * 32) k_gemv_tq2(GemvArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kOpBytes = kOpUnits * kUnitBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                       // CW * NOPS
  uint8_t* ring = smem + ((CW * NOPS * 8 + 127) / 128) * 128;                // CW * NOPS * kOpBytes
  float* csm = reinterpret_cast<float*>(ring + CW * NOPS * kOpBytes);       // KBs x 8NT
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int slice = blockIdx.x / a.cps, cta_in_slice = blockIdx.x % a.cps;
  const int kb0 = (int)((int64_t)slice * a.nb / a.ks), kb1 = (int)((int64_t)(slice + 1) * a.nb / a.ks);
  const int KBs = kb1 - kb0;
  uint8_t* xs = reinterpret_cast<uint8_t*>(csm) + ((KBs * 8 * NT * 4 + 15) / 16) * 16;
  const int units = a.n_tiles * KBs;
  const int W = a.cps * CW;
  const int wi = cta_in_slice * CW + warp;
  const int u_begin = Split<CW>::u0(wi, units, W), u_end = Split<CW>::u0(wi + 1, units, W);
  const int nrows_x = a.batch < 8 * NT ? a.batch : 8 * NT;
  uint64_t* mybar = bars + warp * NOPS;
  uint8_t* myring = ring + warp * NOPS * kOpBytes;
  // an op fetches up to kOpUnits consecutive units of one tile's K-slice run (contiguous bytes)
  auto op_len = [&](int u) {
    int n = u_end - u;
    const int run = KBs - u % KBs;
    if (run < n) n = run;
    return n < kOpUnits ? n : kOpUnits;
  };
  auto op_src = [&](int u) { return a.w + ((int64_t)(u / KBs) * a.nb + kb0 + u % KBs) * kUnitBytes; };

  uint64_t* tsb = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(a.ws) + (32 << 20)) + (size_t)(blockIdx.x * CW + warp) * 8;
  const bool trace = (a.dbg & 4) && lane == 0;
  if (trace) tsb[0] = gtimer();
  // ---- ring setup + prologue prefetch (weights do not depend on the previous kernel)
  int iu = u_begin;   // next unit to fetch (meaningful in lane 0)
  uint64_t pol = 0;
  if (lane == 0) {
    pol = policy_evict_first();
#pragma unroll
    for (int s = 0; s < NOPS; ++s) mbar_init(&mybar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
    for (int s = 0; s < NOPS; ++s) {
      if (iu < u_end) {
        const int n = op_len(iu);
        mbar_expect_tx(&mybar[s], n * kUnitBytes);
        bulk_g2s(myring + s * kOpBytes, op_src(iu), n * kUnitBytes, &mybar[s], pol);
        iu += n;
      }
    }
  }
  __syncwarp();
  griddep_launch_dependents();
  griddep_wait();   // x (and the workspace) belong to the previous kernel until here
  if (trace) tsb[1] = gtimer();

  // ---- stage x[0:nrows_x, kb0*256 : kb1*256) (+ zero row) and the per-block corrections C
  const int xrs = a.xrs;
  for (int i = threadIdx.x; i < xrs / 16; i += blockDim.x)
    *reinterpret_cast<uint4*>(xs + nrows_x * xrs + i * 16) = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < KBs * 8 * NT; i += blockDim.x) csm[i] = 0.0f;
  __syncthreads();
  {
    const T* xg = reinterpret_cast<const T*>(a.x);
    const int64_t kbase = (int64_t)kb0 * kBlock;
    const int xunits = nrows_x * KBs * 32;   // 16-byte units; 32 per (n, block) = one warp
    constexpr int kB = 8;
    for (int base = 0; base < xunits; base += kB * blockDim.x) {
      uint4 v[kB];
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int u = base + i * blockDim.x + threadIdx.x;
        if (u < xunits) {
          const int n = u / (KBs * 32), rem = u % (KBs * 32);
          const int64_t k = kbase + (rem >> 5) * kBlock + (rem & 31) * 8;
          if (a.x_vec && k + 8 <= a.cols) {
            v[i] = *reinterpret_cast<const uint4*>(xg + n * a.ldx + k);
          } else {
            T tmp[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) tmp[e] = (k + e < a.cols) ? xg[n * a.ldx + k + e] : Act<T>::from_float(0.0f);
            v[i] = *reinterpret_cast<uint4*>(tmp);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int u = base + i * blockDim.x + threadIdx.x;
        if (u < xunits) {   // warp-uniform
          const int n = u / (KBs * 32), rem = u % (KBs * 32);
          const int blk = rem >> 5, cu = rem & 31, ch = cu >> 3, q = cu & 7;
          // columns 8q..8q+3 are field class (2q)&3, 8q+4..8q+7 class (2q+1)&3
          const int ja = (2 * q) & 3, jb = ja + 1;
          const float fa = Frag<T>::kFactor(ja), fb = Frag<T>::kFactor(jb);
          uint4 sv4;
          sv4.x = Frag<T>::scale2(v[i].x, fa);
          sv4.y = Frag<T>::scale2(v[i].y, fa);
          sv4.z = Frag<T>::scale2(v[i].z, fb);
          sv4.w = Frag<T>::scale2(v[i].w, fb);
          *reinterpret_cast<uint4*>(xs + n * xrs + blk * kXBlockBytes + ch * kXChunkBytes + q * 16) = sv4;
          float cv = sum4<T>(v[i].x, v[i].y) * (1.0f + Frag<T>::kBase * fa * Frag<T>::kInvF) +
                     sum4<T>(v[i].z, v[i].w) * (1.0f + Frag<T>::kBase * fb * Frag<T>::kInvF);
#pragma unroll
          for (int o = 16; o; o >>= 1) cv += __shfl_xor_sync(0xffffffffu, cv, o);
          if (cu == 0) csm[blk * 8 * NT + n] = cv;
        }
      }
    }
  }
  __syncthreads();
  if (trace) tsb[2] = gtimer();

  const uint8_t* xrow[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int n = 8 * t + g;
    xrow[t] = xs + (n < nrows_x ? n : nrows_x) * xrs + c * kXChunkBytes;
  }

  T* y = reinterpret_cast<T*>(a.y);
  float acc[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[t][e] = 0.0f;
  int cur_tile = u_begin < u_end ? u_begin / KBs : -1;

  auto store_tile = [&](int tile, const float (&v)[NT][4]) {
    const int r0 = tile * 16 + g, r1 = r0 + 8;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int n0 = 8 * t + 2 * c, n1 = n0 + 1;
      if (n0 < a.batch) {
        if (r0 < a.rows) y[n0 * a.ldy + r0] = Act<T>::from_float(v[t][0]);
        if (r1 < a.rows) y[n0 * a.ldy + r1] = Act<T>::from_float(v[t][2]);
      }
      if (n1 < a.batch) {
        if (r0 < a.rows) y[n1 * a.ldy + r0] = Act<T>::from_float(v[t][1]);
        if (r1 < a.rows) y[n1 * a.ldy + r1] = Act<T>::from_float(v[t][3]);
      }
    }
  };
  auto nseg_of = [&](int tile, int s2) {
    const int k0 = (int)((int64_t)s2 * a.nb / a.ks), k1 = (int)((int64_t)(s2 + 1) * a.nb / a.ks);
    const int KB2 = k1 - k0, units2 = a.n_tiles * KB2;
    return Split<CW>::owner(tile * KB2 + KB2 - 1, units2, W) - Split<CW>::owner(tile * KB2, units2, W) + 1;
  };
  // a tile processed entirely by this warp (single K slice) is stored directly
  auto is_whole = [&](int tile) {
    return a.ks == 1 && Split<CW>::owner(tile * KBs, units, W) == wi &&
           Split<CW>::owner(tile * KBs + KBs - 1, units, W) == wi;
  };
  // partial segment: workspace + arrival counter; the last arriver reduces all
  // segments of the tile in a fixed (slice, warp) order and stores y.
  auto flush_part = [&](int tile, const float (&v)[NT][4]) {
    const int first = Split<CW>::owner(tile * KBs, units, W);
    constexpr int kSegFloats = NT * 4 * 32;
    const int seg = slice * a.segs_per_slice + (wi - first);
    float* dst = a.ws + ((int64_t)tile * a.ks * a.segs_per_slice + seg) * kSegFloats;
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) __stcg(dst + (t * 4 + e) * 32 + lane, v[t][e]);
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      int total = 0;
      for (int s2 = 0; s2 < a.ks; ++s2) total += nseg_of(tile, s2);
      const int prev = atomicAdd(a.counters + tile, 1);
      last = (prev == total - 1);
      if (last) a.counters[tile] = 0;   // self-reset for the next launch
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();
    float sum[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) sum[t][e] = 0.0f;
    for (int s2 = 0; s2 < a.ks; ++s2) {
      const int nseg = nseg_of(tile, s2);
      const float* src = a.ws + ((int64_t)tile * a.ks * a.segs_per_slice + s2 * a.segs_per_slice) * kSegFloats;
      int q = 0;
      for (; q + 4 <= nseg; q += 4) {   // four segments' loads in flight at once
        float vv[4][NT][4];
#pragma unroll
        for (int z = 0; z < 4; ++z)
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) vv[z][t][e] = __ldcg(src + (q + z) * kSegFloats + (t * 4 + e) * 32 + lane);
#pragma unroll
        for (int z = 0; z < 4; ++z)
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) sum[t][e] += vv[z][t][e];
      }
      for (; q < nseg; ++q)
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) sum[t][e] += __ldcg(src + q * kSegFloats + (t * 4 + e) * 32 + lane);
    }
    store_tile(tile, sum);
  };
  // The warp's leading partial tile is stashed and flushed at the end, so the
  // fence/atomic latency never stalls the weight stream mid-range.
  int stash_tile = -1;
  float stash[NT][4];
  auto close_tile = [&](int tile) {
    if (is_whole(tile)) {
      store_tile(tile, acc);
    } else if (stash_tile < 0 && tile == u_begin / KBs) {
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) stash[t][e] = acc[t][e];
      stash_tile = tile;
    } else {
      flush_part(tile, acc);
    }
  };

  int u = u_begin, k = 0;
  while (u < u_end) {
    const int n = op_len(u);
    const int s = k % NOPS;
    mbar_wait(&mybar[s], (k / NOPS) & 1);
    if (trace && k == 0) tsb[3] = gtimer();
    const uint8_t* slot = myring + s * kOpBytes;
    uint4 wl[kOpUnits], wh[kOpUnits];
    uint32_t sv[kOpUnits];
#pragma unroll
    for (int q = 0; q < kOpUnits; ++q) {
      if (q < n) {
        wl[q] = *reinterpret_cast<const uint4*>(slot + q * kUnitBytes + (c * 8 + g) * 16);
        wh[q] = *reinterpret_cast<const uint4*>(slot + q * kUnitBytes + 512 + (c * 8 + g) * 16);
        sv[q] = *reinterpret_cast<const uint32_t*>(slot + q * kUnitBytes + kTileBlockBytes + g * 4);
      }
    }
    __syncwarp();
    if (lane == 0 && iu < u_end) {   // refill this slot with the next op
      const int nn = op_len(iu);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_tx(&mybar[s], nn * kUnitBytes);
      bulk_g2s(myring + s * kOpBytes, op_src(iu), nn * kUnitBytes, &mybar[s], pol);
      iu += nn;
    }
#pragma unroll
    for (int q = 0; q < kOpUnits; ++q) {
      if (q < n) {
        const int uu = u + q;
        const int tile = uu / KBs, kl = uu % KBs;
        if (tile != cur_tile) {
          close_tile(cur_tile);
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[t][e] = 0.0f;
          cur_tile = tile;
        }
        if (a.dbg & 1) {
          acc[0][0] += __uint_as_float(wl[q].x ^ wh[q].y ^ sv[q]);
          continue;
        }
        float P[NT][4];
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) P[t][e] = 0.0f;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint32_t L0 = p ? wl[q].z : wl[q].x, L1 = p ? wl[q].w : wl[q].y;
          const uint32_t H0 = p ? wh[q].z : wh[q].x, H1 = p ? wh[q].w : wh[q].y;
          const uint32_t L08 = L0 >> 8, L18 = L1 >> 8, H08 = H0 >> 8, H18 = H1 >> 8;
#pragma unroll
          for (int hb = 0; hb < 2; ++hb) {
            uint4 xv[NT][2];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const uint8_t* xp = xrow[t] + kl * kXBlockBytes + (4 * p + 2 * hb) * 16;
              xv[t][0] = *reinterpret_cast<const uint4*>(xp);
              xv[t][1] = *reinterpret_cast<const uint4*>(xp + 16);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t A[4] = {Frag<T>::field(L0, L08, hb, j), Frag<T>::field(H0, H08, hb, j),
                                     Frag<T>::field(L1, L18, hb, j), Frag<T>::field(H1, H18, hb, j)};
#pragma unroll
              for (int t = 0; t < NT; ++t) {
                const uint4& xx = xv[t][j >> 1];
                Frag<T>::mma(P[t], A, (j & 1) ? xx.z : xx.x, (j & 1) ? xx.w : xx.y);
              }
            }
          }
        }
        const __half2 sp2 = *reinterpret_cast<const __half2*>(&sv[q]);
        const float s_lo = __low2float(sp2), s_hi = __high2float(sp2);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const float2 cc = *reinterpret_cast<const float2*>(csm + kl * 8 * NT + 8 * t + 2 * c);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float yb = fmaf(Frag<T>::kInvF, P[t][e], -((e & 1) ? cc.y : cc.x));
            acc[t][e] = fmaf((e & 2) ? s_hi : s_lo, yb, acc[t][e]);
          }
        }
      }
    }
    u += n;
    ++k;
  }
  if (trace) tsb[4] = gtimer();
  if (stash_tile >= 0) flush_part(stash_tile, stash);
  if (cur_tile >= 0) {
    if (is_whole(cur_tile)) store_tile(cur_tile, acc);
    else flush_part(cur_tile, acc);
  }
  if (trace) tsb[5] = gtimer();
}

// ------------------------------------------------------------------------------------ host

constexpr int kCW = 8;          // warps per CTA
constexpr int kNOPS = 2;        // in-flight bulk copies (4 units each) per warp
constexpr int kXBudget = 48 * 1024;
constexpr size_t kCounterBytes = 256 * 1024;   // per-tile arrival counters: up to 65536 tiles (1M rows)

struct GemvPlan {
  int ks, cps, segs_per_slice, xrs, nrows_x, nt;
  size_t smem, ws_floats;
  int n_tiles, nb;
};

static GemvPlan plan_gemv(int batch, int rows, int cols, int ks_force, int sm_count) {
  GemvPlan p;
  p.nb = (int)ceil_div(cols, kBlock);
  p.n_tiles = (int)(rows_padded(rows) / 16);
  p.nt = batch <= 8 ? 1 : (batch <= 16 ? 2 : 4);
  p.nrows_x = batch < 8 * p.nt ? batch : 8 * p.nt;
  int ks = ks_force > 0 ? ks_force : 1;
  if (ks_force <= 0)
    while (ks < p.nb && (int64_t)(p.nrows_x + 1) * x_row_stride((int)ceil_div(p.nb, ks)) > kXBudget) ++ks;
  if (ks > p.nb) ks = p.nb;
  p.ks = ks;
  const int kbmax = (int)ceil_div(p.nb, ks), kbmin = p.nb / ks;
  const int64_t units_min = (int64_t)p.n_tiles * kbmin;
  // CTAs per slice: fill 2 CTAs/SM, but give each warp >= 4 units (one full bulk copy)
  int cps = (2 * sm_count) / ks;
  if (cps < 1) cps = 1;
  const int64_t by_work = ceil_div(units_min, 4 * kCW);
  if (cps > by_work) cps = (int)(by_work > 0 ? by_work : 1);
  p.cps = cps;
  const int64_t W = (int64_t)cps * kCW;
  const int64_t lmin = units_min / W;   // >= 1 unless tiny
  p.segs_per_slice = (int)(lmin >= 1 ? (kbmax - 1) / lmin + 2 : kbmax + 1);
  p.xrs = x_row_stride(kbmax);
  p.smem = (size_t)((kCW * kNOPS * 8 + 127) / 128) * 128 + (size_t)kCW * kNOPS * kOpUnits * kUnitBytes + ((size_t)kbmax * 8 * p.nt * 4 + 15) / 16 * 16 +
           (size_t)(p.nrows_x + 1) * p.xrs;
  p.ws_floats = (size_t)p.n_tiles * ks * p.segs_per_slice * p.nt * 4 * 32;
  return p;
}

static int sm_count_cached() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

size_t gemv_workspace_bytes(int batch, int rows, int cols) {
  const int b = batch < 32 ? batch : 32;
  GemvPlan p = plan_gemv(b > 0 ? b : 1, rows, cols, 0, 148);
  // counters first (a fixed region, so shapes sharing a workspace never see each
  // other's partial sums in their counters), then partial segments
  size_t cnt = kCounterBytes;
  // worst case over ks choices the caller may force: size for ks up to 8
  GemvPlan p8 = plan_gemv(b > 0 ? b : 1, rows, cols, 8, 148);
  size_t ws = p.ws_floats > p8.ws_floats ? p.ws_floats : p8.ws_floats;
  return cnt + ws * 4 * 2;
}

template <typename T, int NT>
static int launch_gemv(GemvArgs a, const GemvPlan& p, int pdl, cudaStream_t st) {
  auto kern = k_gemv_tq2<T, NT, kCW, kNOPS>;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured_dev = dev;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.ks * p.cps, 1, 1);
  cfg.blockDim = dim3(kCW * 32, 1, 1);
  cfg.dynamicSmemBytes = p.smem;
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) {
    set_error("tr_linear(gemv): launch failed: %s (grid %d, smem %zu, ks %d)", cudaGetErrorString(e),
              (int)cfg.gridDim.x, p.smem, p.ks);
    return -1;
  }
  return 0;
}

int gemv_tq2(int act, const void* w, const void* x, void* y, int64_t ldx, int64_t ldy, int batch, int rows,
             int cols, int ks, void* workspace, size_t ws_bytes, int pdl, int dbg, cudaStream_t st) {
  GemvPlan p = plan_gemv(batch, rows, cols, ks, sm_count_cached());
  const size_t cnt = kCounterBytes;
  if ((size_t)p.n_tiles * 4 > kCounterBytes) {
    set_error("tr_linear: %d row tiles exceed the workspace counter region", p.n_tiles);
    return -1;
  }
  if (workspace == nullptr || ws_bytes < cnt + p.ws_floats * 4) {
    set_error("tr_linear: workspace too small (%zu < %zu bytes); size it with tr_linear_workspace_size", ws_bytes,
              cnt + p.ws_floats * 4);
    return -1;
  }
  GemvArgs a;
  a.w = (const uint8_t*)w;
  a.x = x;
  a.y = y;
  a.counters = (int*)workspace;
  a.ws = (float*)((uint8_t*)workspace + cnt);
  a.ldx = ldx;
  a.ldy = ldy;
  a.rows = rows;
  a.cols = cols;
  a.nb = p.nb;
  a.n_tiles = p.n_tiles;
  a.batch = batch;
  a.ks = p.ks;
  a.cps = p.cps;
  a.segs_per_slice = p.segs_per_slice;
  a.xrs = p.xrs;
  a.x_vec = ((ldx % 8) == 0 && ((uintptr_t)x % 16) == 0) ? 1 : 0;
  a.dbg = dbg;
  if (act == kActF16) {
    if (p.nt == 1) return launch_gemv<__half, 1>(a, p, pdl, st);
    if (p.nt == 2) return launch_gemv<__half, 2>(a, p, pdl, st);
    return launch_gemv<__half, 4>(a, p, pdl, st);
  }
  if (p.nt == 1) return launch_gemv<__nv_bfloat16, 1>(a, p, pdl, st);
  if (p.nt == 2) return launch_gemv<__nv_bfloat16, 2>(a, p, pdl, st);
  return launch_gemv<__nv_bfloat16, 4>(a, p, pdl, st);
}

}  // namespace tr
