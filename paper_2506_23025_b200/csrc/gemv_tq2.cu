// K3: decode-side ternary GEMV / skinny GEMM (batch 1..32), TQ2 weights.
//
// Semantics (reference linear.py:137-166, _kernels.pyx:136-168; paper App. F):
//   y[n, r] = sum_b s[r, b] * (sum_{k in block b} trit[r, k] * x[n, k])
// fp16/bf16 activations; each 256-block's inner sum is accumulated in fp32,
// multiplied by the fp32 value of its binary16 scale and added to an fp32 row
// accumulator; the output is rounded once (RNE).
//
// B200 design: the kernel is a short latency chain, because a
// decode layer moves only 4-60 MB (0.7-9 us of HBM time):
//  * one CTA per SM owns a contiguous run of whole 16-row tiles (all K), so no
//    result ever crosses CTAs -- no global atomics, fences or fix-up passes;
//  * the CTA's weights are one contiguous byte range of the T16 layout, pulled
//    through an R-slot shared-memory ring of 8-unit chunks by cp.async.bulk
//    (TMA bulk copies completing on mbarriers).  The first R copies are issued
//    before griddepcontrol.wait, so a PDL-chained layer streams its weights while
//    the previous layer finishes (smem is sized so two layers co-reside per SM);
//    the last warp to release a slot refills it -- no producer warp;
//  * warp w takes unit w of every chunk (K-split of each tile across warps);
//    decode is one LOP3 per half2 (fp16: digit * 4^j * 2^-24 subnormal; bf16:
//    128 + digit * m_j) feeding mma.sync.m16n8k16 A fragments, one fp32
//    accumulator per field class j; B fragments come straight from x (L1);
//    sum (d-1) x = sum_j P_j / F_j - C with C = sum x per (block, row) computed
//    once per CTA (which also warms L1 with x);
//  * a warp leaving a tile deposits its fragment in a shared slot; the last of
//    the tile's warps sums the fragments in fixed warp order and stores y --
//    deterministic, and no CTA-wide barrier in the main loop.
#include <vector>

#include "common.cuh"

namespace tr {

#ifndef GEMV_SU1
#define GEMV_SU1 4
#endif
#ifndef GEMV_NSMAX
#define GEMV_NSMAX 4
#endif
constexpr int kNSMax = GEMV_NSMAX;     // ring slots per warp at 2 units per slot (a power of two; fewer when the range is short)
constexpr int kXChunk = 144;   // staged activations: bytes per 64-column chunk (128 + bank spread)
constexpr int kXBlk = 4 * kXChunk;

template <typename T> struct Frag;
template <> struct Frag<__half> {
  // exponent field left zero: a field is the subnormal d * 4^j * 2^-24 (base 0)
  __device__ static float inv_f(int j) {
    return j == 0 ? 16777216.0f : j == 1 ? 4194304.0f : j == 2 ? 1048576.0f : 262144.0f;
  }
  static constexpr float kBase = 0.0f;
  __device__ static uint32_t field(uint32_t w, uint32_t w8, int hb, int j) {
    return (hb ? w8 : w) & (0x00030003u << (2 * j));
  }
  __device__ static void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  __device__ static float2 to_f2(uint32_t v) { return __half22float2(*reinterpret_cast<const __half2*>(&v)); }
};
template <> struct Frag<__nv_bfloat16> {
  // magic exponent 0x4300 (128.0): a field is 128 + m_j * d, m_j = 4^j (j < 3), m_3 = 1
  __device__ static float inv_f(int j) { return j == 0 ? 1.0f : j == 1 ? 0.25f : j == 2 ? 0.0625f : 1.0f; }
  static constexpr float kBase = 128.0f;
  __device__ static uint32_t field(uint32_t w, uint32_t w8, int hb, int j) {
    if (j < 3) return ((hb ? w8 : w) & (0x00030003u << (2 * j))) | 0x43004300u;
    return ((w >> (hb ? 14 : 6)) & 0x00030003u) | 0x43004300u;
  }
  __device__ static void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  __device__ static float2 to_f2(uint32_t v) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v));
  }
};

struct GemvLayer {    // one product y = x W^T (the C-ABI's TrStackLayer, plus derived sizes)
  const uint8_t* w;   // T16 units, tile-major
  const void* x;      // [batch][ldx]
  void* y;            // [batch][ldy]
  int64_t ldx, ldy;
  int rows, cols, nb, n_tiles;
  int x_vec;          // x rows 16-byte aligned
  int pad_;
};

struct GemvArgs {
  GemvLayer l0;                  // the layer (single product), or unused
  const GemvLayer* layers;       // device layer table for a persistent chain (nullptr: just l0)
  unsigned* bar;                 // grid barrier {count, generation} (chain only; zero-initialised)
  int n_layers;
  int nb_max;                    // shared-memory layout is sized for the widest layer
  int batch;
  int ns;                        // ring slots per warp
  int dbg;                       // development probe: 2 = per-CTA timestamps into y
  // fused producer of x (decode glue folded into the staging, single layer + XS only):
  // 1: x = rmsnorm(x + delta) * gamma, CTA 0 also stores x + delta to x_out (the residual);
  // 2: x = silu(x[:, :cols]) * x[:, cols:2 cols] (SwiGLU of a gate|up product)
  int pre;
  const void* pre_delta;
  const void* pre_gamma;
  void* pre_out;
  float eps;
  int out_f32;                   // TR_LINEAR_OUT_F32: y is float32
};

// Sense-reversal grid barrier for the persistent chain (all CTAs are co-resident: the
// chain is launched cooperatively).  The counter self-resets; the generation only grows.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ uint4 ld_cg_x8(const T* row, int64_t k, int cols, int vec) {   // coherent (L2) path
  if (vec && k + 8 <= cols) return __ldcg(reinterpret_cast<const uint4*>(row + k));
  T tmp[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) tmp[e] = (k + e < cols) ? __ldcg(row + k + e) : Act<T>::from_float(0.0f);
  return *reinterpret_cast<uint4*>(tmp);
}

// Shared-memory plan: [barriers, slot tags | reduction slots | C | staged x | per-warp weight rings].
// NW warps per CTA: 16 (one CTA per SM) for long per-CTA ranges; 8 with <= 128 registers
// so that two CTAs fit per SM and a PDL-chained next layer starts (and prefetches its
// weights) while this one computes -- the better trade for small layers.
template <int NT, int NW> struct GemvCfg {
  static constexpr int kWarps = NW;     // warps per CTA
  static constexpr int kSU = NT == 1 ? GEMV_SU1 : 2;   // units (1056 B) per bulk copy = one ring slot
  static constexpr int kFrag = NT * 4 * 32;            // floats of one warp's tile fragment
  static constexpr int kSlotBytes = kSU * kUnitBytes;
  static constexpr size_t kRedOff = 1024;
  static constexpr size_t kCsumOff = kRedOff + (size_t)2 * kWarps * kFrag * 4;
  // staged x row: per 256-block 4 chunks of 64 halves at a 144-byte pitch (the 4 chunks a
  // B-fragment load touches sit in different banks), row pitch == 64 (mod 128)
  __host__ __device__ static int x_stride(int nb) { return nb * kXBlk + ((nb & 1) ? 0 : 64); }
  __host__ __device__ static size_t xs_off(int nb) { return kCsumOff + ((size_t)nb * 8 * NT * 4 + 15) / 16 * 16; }
  __host__ __device__ static size_t ring_off(int nb, int nrx, bool xs) {
    return (xs_off(nb) + (xs ? (size_t)nrx * x_stride(nb) : 0) + 127) / 128 * 128;
  }
  __host__ __device__ static size_t smem(int nb, int nrx, bool xs, int ns) {
    return ring_off(nb, nrx, xs) + (size_t)kWarps * ns * kSlotBytes;
  }
};

// 8 consecutive activations x[row][k..k+7] (zero past cols), read through L1
template <typename T>
__device__ __noinline__ uint4 load_x8_slow(const T* row, int64_t k, int cols) {
  T tmp[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) tmp[e] = (k + e < cols) ? row[k + e] : Act<T>::from_float(0.0f);
  return *reinterpret_cast<uint4*>(tmp);
}
template <typename T>
__device__ __forceinline__ uint4 load_x8(const T* row, int64_t k, int cols, int vec) {
  if (vec && k + 8 <= cols) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(row + k));
    return r;
  }
  return load_x8_slow(row, k, cols);
}

// XS: activations staged in shared memory (when they fit), else read through L1
__device__ __forceinline__ float tof(__half v) { return __half2float(v); }
__device__ __forceinline__ float tof(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ void f8_from(const uint4& v, float (&f)[8]) {
  const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = tof(e[i]);
}
template <typename T>
__device__ __forceinline__ uint4 f8_to(const float (&f)[8]) {
  uint4 v;
  T* e = reinterpret_cast<T*>(&v);
#pragma unroll
  for (int i = 0; i < 8; ++i) e[i] = Act<T>::from_float(f[i]);
  return v;
}
template <typename T>
__device__ __forceinline__ float rnd(float v) { return tof(Act<T>::from_float(v)); }   // round through T

// Fused decode glue (GemvArgs::pre): writes the producer's output straight into the
// staged-activation buffer xs (same arithmetic and roundings as tr_add_rmsnorm /
// tr_silu_mul).  scratch: >= nb * 8 floats (the boundary-reduction buffer, free here).
template <typename T, typename Ly_t>
__device__ void stage_pre(const GemvArgs& a, const Ly_t& Ly, uint8_t* xs, int rs, float* scratch, int nrx) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nb = Ly.nb, cols = Ly.cols;
  const T* xg = reinterpret_cast<const T*>(Ly.x);
  auto at = [&](int n, int kb) { return xs + n * rs + kb * kXBlk + (lane >> 3) * kXChunk + (lane & 7) * 16; };
  for (int item = warp; item < nb * nrx; item += nw) {
    const int kb = item / nrx, n = item % nrx;
    const int64_t kx = (int64_t)kb * kBlock + lane * 8;
    float f[8];
    if (a.pre == 2) {   // silu(gate) * up
      float g[8], u[8];
      f8_from<T>(load_x8(xg + n * Ly.ldx, kx, cols, Ly.x_vec), g);
      f8_from<T>(load_x8(xg + n * Ly.ldx + cols, kx, cols, Ly.x_vec), u);
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = rnd<T>(__fdividef(g[e], 1.0f + __expf(-g[e]))) * u[e];   // (0 past cols)
      *reinterpret_cast<uint4*>(at(n, kb)) = f8_to<T>(f);
    } else {            // residual add, stored rounded; sum of squares per (block, row)
      f8_from<T>(load_x8(xg + n * Ly.ldx, kx, cols, Ly.x_vec), f);
      if (a.pre_delta) {
        float d[8];
        f8_from<T>(load_x8(reinterpret_cast<const T*>(a.pre_delta) + n * Ly.ldx, kx, cols, Ly.x_vec), d);
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = rnd<T>(f[e] + d[e]);
      }
      const uint4 hv = f8_to<T>(f);
      *reinterpret_cast<uint4*>(at(n, kb)) = hv;
      if (blockIdx.x == 0 && a.pre_out && kx < cols) {
        T* o = reinterpret_cast<T*>(a.pre_out) + n * Ly.ldx + kx;
        if (kx + 8 <= cols && Ly.x_vec) {
          *reinterpret_cast<uint4*>(o) = hv;
        } else {
          const T* he = reinterpret_cast<const T*>(&hv);
          for (int e = 0; e < 8 && kx + e < cols; ++e) o[e] = he[e];
        }
      }
      float ss = 0.0f;
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += f[e] * f[e];
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) scratch[kb * 8 + n] = ss;
    }
  }
  __syncthreads();
  if (a.pre != 1) return;
  float* inv = scratch + nb * 8;   // per row: rsqrt(mean(h^2) + eps), fixed-order sums
  for (int n = warp; n < nrx; n += nw) {
    float ss = 0.0f;
    for (int kb = lane; kb < nb; kb += 32) ss += scratch[kb * 8 + n];
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) inv[n] = rsqrtf(ss / cols + a.eps);
  }
  __syncthreads();
  const T* gam = reinterpret_cast<const T*>(a.pre_gamma);
  for (int item = warp; item < nb * nrx; item += nw) {
    const int kb = item / nrx, n = item % nrx;
    const int64_t kx = (int64_t)kb * kBlock + lane * 8;
    float f[8], g[8];
    f8_from<T>(*reinterpret_cast<const uint4*>(at(n, kb)), f);
    f8_from<T>(load_x8(gam, kx, cols, Ly.x_vec), g);
    const float iv = inv[n];
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = rnd<T>(f[e] * iv) * g[e];
    *reinterpret_cast<uint4*>(at(n, kb)) = f8_to<T>(f);
  }
  __syncthreads();
}

template <typename T, int NT, bool XS, int NW>
__global__ void __launch_bounds__(NW * 32, (NW == 8 && NT == 1) ? 2 : 1) k_gemv_tq2(const GemvArgs a) {
  using Cfg = GemvCfg<NT, NW>;
  constexpr int kFrag = Cfg::kFrag, kWarps = Cfg::kWarps, kSlotBytes = Cfg::kSlotBytes, kSU = Cfg::kSU;
  const int NS = a.ns;
  extern __shared__ __align__(128) uint8_t smem[];
  const int nrx = a.batch < 8 * NT ? a.batch : 8 * NT;
  const bool chain = a.layers != nullptr;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                      // kWarps * NS (<= 64)
  int* slot_tile = reinterpret_cast<int*>(smem + 512);                      // 2 * kWarps
  float* red = reinterpret_cast<float*>(smem + Cfg::kRedOff);               // 2 * kWarps * kFrag
  float* csum = reinterpret_cast<float*>(smem + Cfg::kCsumOff);             // nb x 8NT
  uint8_t* xs = smem + Cfg::xs_off(a.nb_max);                               // XS: nrx x x_stride
  uint8_t* ring = smem + Cfg::ring_off(a.nb_max, nrx, XS);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  uint64_t* mybar = bars + warp * NS;
  uint8_t* myring = ring + warp * NS * kSlotBytes;
  auto layer = [&](int l) -> GemvLayer { return chain ? a.layers[l] : a.l0; };
  // the CTA owns whole tiles [t0, t1) of a layer; warp w a contiguous slice of its units
  auto warp_range = [&](const GemvLayer& L_, int& u0, int& u1) {
    const int t0 = (int)((int64_t)blockIdx.x * L_.n_tiles / gridDim.x);
    const int t1 = (int)((int64_t)(blockIdx.x + 1) * L_.n_tiles / gridDim.x);
    const int cu0 = t0 * L_.nb, LL = (t1 - t0) * L_.nb;
    u0 = cu0 + (int)((int64_t)warp * LL / kWarps);
    u1 = cu0 + (int)((int64_t)(warp + 1) * LL / kWarps);
  };
  uint64_t* trace = (a.dbg & 2) ? reinterpret_cast<uint64_t*>(a.l0.y) + blockIdx.x * 8 : nullptr;
  auto stamp = [&](int k) {
    if (trace && threadIdx.x == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      trace[k] = t;
    }
  };
  stamp(0);

  // ---- weight producer (lane 0): one op stream over every layer's range, so the ring keeps
  // prefetching the next layer's weights (they do not depend on x) across layer boundaries
  int pl = 0, pu = 0, pu1 = 0;   // producer: layer, next unit, end of this warp's range
  const uint8_t* pw = nullptr;
  uint64_t pol = 0;
  auto producer_seek = [&]() {     // advance to the next layer with a non-empty range
    while (pu >= pu1 && pl < a.n_layers) {
      if (++pl < a.n_layers) {
        const GemvLayer L_ = layer(pl);
        warp_range(L_, pu, pu1);
        pw = L_.w;
      }
    }
  };
  auto issue = [&](int slot) -> bool {   // lane 0: next op into `slot`; false when the stream is done
    if (pl >= a.n_layers) return false;
    const int n = min(kSU, pu1 - pu);
    mbar_expect_tx(&mybar[slot], n * kUnitBytes);
    bulk_g2s(myring + slot * kSlotBytes, pw + (int64_t)pu * kUnitBytes, n * kUnitBytes, &mybar[slot], pol);
    pu += n;
    producer_seek();
    return true;
  };
  if (lane == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < NS; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
    const GemvLayer L0 = layer(0);
    warp_range(L0, pu, pu1);
    pw = L0.w;
    pl = 0;
    producer_seek();   // (skips layers where this warp has no units)
    for (int s = 0; s < NS; ++s)
      if (!issue(s)) break;
  }
  __syncwarp();
  griddep_launch_dependents();
  griddep_wait();   // x belongs to the previous kernel until here
  stamp(1);

  int k = 0;   // consumer op counter (ring slot k % NS)
  const int nslog = NS == 1 ? 0 : NS == 2 ? 1 : 2;   // NS is a power of two (host)
  float acc[NT][4];
  float P[4][NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc[t][e] = 0.0f;
#pragma unroll
      for (int j = 0; j < 4; ++j) P[j][t][e] = 0.0f;
    }

  for (int l = 0; l < a.n_layers; ++l) {
    const GemvLayer Ly = layer(l);
    const int nb = Ly.nb;
    if (l > 0) grid_barrier(a.bar);   // every CTA has stored layer l-1's y (= this layer's x)
    if (lane == 0) {
      slot_tile[2 * warp] = -1;
      slot_tile[2 * warp + 1] = -1;
    }
    // ---- per-(block, row) correction C = sum_k x_k (1 + base / m_j(k)); stages x (XS) or warms L1
    const T* xg = reinterpret_cast<const T*>(Ly.x);
    const int rs = Cfg::x_stride(nb);
    if (XS && a.pre) stage_pre<T>(a, Ly, xs, rs, red, nrx);   // fused glue: xs already holds x
    for (int item = warp; item < nb * nrx; item += kWarps) {
      const int kb = item / nrx, n = item % nrx;
      const int64_t kx = (int64_t)kb * kBlock + lane * 8;
      uint4 v;
      uint8_t* xsp = xs + n * rs + kb * kXBlk + (lane >> 3) * kXChunk + (lane & 7) * 16;
      if (XS && a.pre) {
        v = *reinterpret_cast<const uint4*>(xsp);
      } else {
        v = chain ? ld_cg_x8(xg + n * Ly.ldx, kx, Ly.cols, Ly.x_vec) : load_x8(xg + n * Ly.ldx, kx, Ly.cols, Ly.x_vec);
        if (XS) *reinterpret_cast<uint4*>(xsp) = v;
      }
      // chunk column (8 lane + e) % 64 has field class j = (col >> 2) & 3
      const int ja = (2 * lane) & 3, jb = ja + 1;
      const float fa = 1.0f + Frag<T>::kBase * Frag<T>::inv_f(ja), fb = 1.0f + Frag<T>::kBase * Frag<T>::inv_f(jb);
      const float2 p0 = Frag<T>::to_f2(v.x), p1 = Frag<T>::to_f2(v.y), p2 = Frag<T>::to_f2(v.z),
                   p3 = Frag<T>::to_f2(v.w);
      float sm = ((p0.x + p0.y) + (p1.x + p1.y)) * fa + ((p2.x + p2.y) + (p3.x + p3.y)) * fb;
#pragma unroll
      for (int o = 16; o; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
      if (lane == 0) csum[kb * 8 * NT + n] = sm;
    }
    __syncthreads();
    stamp(2);

    int wu0, wu1;
    warp_range(Ly, wu0, wu1);
    T* y = reinterpret_cast<T*>(Ly.y);
    auto store_tile = [&](int tile, const float (&v)[NT][4]) {
      if (trace) return;
      const int r0 = tile * 16 + g, r1 = r0 + 8;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int n0 = 8 * t + 2 * c, n1 = n0 + 1;
        if (n0 < a.batch) {
          if (r0 < Ly.rows) store_y<T>(Ly.y, (int64_t)n0 * Ly.ldy + r0, v[t][0], a.out_f32);
          if (r1 < Ly.rows) store_y<T>(Ly.y, (int64_t)n0 * Ly.ldy + r1, v[t][2], a.out_f32);
        }
        if (n1 < a.batch) {
          if (r0 < Ly.rows) store_y<T>(Ly.y, (int64_t)n1 * Ly.ldy + r0, v[t][1], a.out_f32);
          if (r1 < Ly.rows) store_y<T>(Ly.y, (int64_t)n1 * Ly.ldy + r1, v[t][3], a.out_f32);
        }
      }
    };
    const int first_tile = wu0 < wu1 ? wu0 / nb : -1;
    int cur = first_tile;
    // a tile wholly inside this warp's range is stored now; a boundary tile is parked
    // in a reduction slot (0: the warp's first tile, 1: its last) and combined below
    auto close_tile = [&](int tile) {
      if (tile * nb >= wu0 && (tile + 1) * nb <= wu1) {
        store_tile(tile, acc);
        return;
      }
      const int which = (tile == first_tile) ? 0 : 1;
      float* dst = red + (2 * warp + which) * kFrag;
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) dst[(t * 4 + e) * 32 + lane] = acc[t][e];
      if (lane == 0) slot_tile[2 * warp + which] = tile;
    };

    // B-fragment rows: lanes past the batch read row 0 -- their output columns are never stored
    const uint8_t* xsrow[NT];
    const T* xrow[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int n = min(8 * t + g, nrx - 1);
      xrow[t] = xg + n * Ly.ldx;
      xsrow[t] = xs + n * rs + c * kXChunk;
    }

    // one 16x256 unit: decode + 16 (x NT) mma.sync, then the block epilogue into acc
    auto do_unit = [&](const uint4& wl, const uint4& wh, uint32_t sv, int kb) {
      const int64_t kx = (int64_t)kb * kBlock + c * 64;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const uint32_t L0 = p ? wl.z : wl.x, L1 = p ? wl.w : wl.y;
        const uint32_t H0 = p ? wh.z : wh.x, H1 = p ? wh.w : wh.y;
        const uint32_t L08 = L0 >> 8, L18 = L1 >> 8, H08 = H0 >> 8, H18 = H1 >> 8;
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          uint4 xv[NT][2];
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (XS) {
              const uint8_t* xp = xsrow[t] + kb * kXBlk + 32 * (2 * p + hb);
              xv[t][0] = lds128(xp);
              xv[t][1] = lds128(xp + 16);
            } else {
              xv[t][0] = load_x8(xrow[t], kx + 16 * (2 * p + hb), Ly.cols, Ly.x_vec);
              xv[t][1] = load_x8(xrow[t], kx + 16 * (2 * p + hb) + 8, Ly.cols, Ly.x_vec);
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t A[4] = {Frag<T>::field(L0, L08, hb, j), Frag<T>::field(H0, H08, hb, j),
                                   Frag<T>::field(L1, L18, hb, j), Frag<T>::field(H1, H18, hb, j)};
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const uint4& xx = xv[t][j >> 1];
              Frag<T>::mma(P[j][t], A, (j & 1) ? xx.z : xx.x, (j & 1) ? xx.w : xx.y);
            }
          }
        }
      }
      // block epilogue: block sum in fp32, times the block scale, into the row accumulator
      const float2 sc = __half22float2(*reinterpret_cast<const __half2*>(&sv));
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const float2 cv = *reinterpret_cast<const float2*>(csum + kb * 8 * NT + 8 * t + 2 * c);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float yb = fmaf(P[0][t][e], Frag<T>::inv_f(0), -((e & 1) ? cv.y : cv.x));
          yb = fmaf(P[1][t][e], Frag<T>::inv_f(1), yb);
          yb = fmaf(P[2][t][e], Frag<T>::inv_f(2), yb);
          yb = fmaf(P[3][t][e], Frag<T>::inv_f(3), yb);
          acc[t][e] = fmaf((e & 2) ? sc.y : sc.x, yb, acc[t][e]);
#pragma unroll
          for (int j = 0; j < 4; ++j) P[j][t][e] = 0.0f;
        }
      }
    };

    int kb = wu0 - (wu0 < wu1 ? first_tile : 0) * nb;   // block of the next unit within tile `cur`
    auto unit = [&](const uint4& wl, const uint4& wh, uint32_t sv) {
      if (kb == nb) {   // next tile
        close_tile(cur);
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[t][e] = 0.0f;
        ++cur;
        kb = 0;
      }
      do_unit(wl, wh, sv, kb);
      ++kb;
    };

    int u = wu0;
#pragma unroll 1
    for (; u < wu1; ++k) {
      const int s = k & (NS - 1);
      const int n = min(kSU, wu1 - u);
      // refill the slot read in the PREVIOUS iteration: its loads have long completed (their
      // values fed the MMAs), so the proxy fence does not stall on outstanding loads
#ifdef GEMV_NOWAIT   // dev probe: compute on the first ring fill only (wrong results; times the math)
      if (k >= NS) goto skip_wait;
#endif
      if (k > 0) {
        __syncwarp();
        if (lane == 0) {
          fence_proxy_async_smem();
          issue((k - 1) & (NS - 1));
        }
      }
      mbar_wait(&mybar[s], (k >> nslog) & 1);
      if (k == 0) stamp(3);
#ifdef GEMV_NOWAIT
    skip_wait:
#endif
      const uint8_t* slot = myring + s * kSlotBytes + t16_word(0, c, g) * 16;
      uint4 wl[kSU], wh[kSU];
      uint32_t sv[kSU];
#pragma unroll
      for (int q = 0; q < kSU; ++q) {
        if (q < n) {
          wl[q] = lds128(slot + q * kUnitBytes);
          wh[q] = lds128(slot + q * kUnitBytes + 512);
          sv[q] = *reinterpret_cast<const uint32_t*>(slot - t16_word(0, c, g) * 16 + q * kUnitBytes + kTileBlockBytes + g * 4);
        }
      }
#pragma unroll
      for (int q = 0; q < kSU; ++q)
        if (q < n) unit(wl[q], wh[q], sv[q]);
      u += n;
    }
    stamp(4);
    if (trace && lane == 0) {   // per-warp loop end (development trace)
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      reinterpret_cast<uint64_t*>(a.l0.y)[148 * 8 + blockIdx.x * 32 + warp] = t;
    }
    if (cur >= 0) close_tile(cur);
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[t][e] = 0.0f;

    // ---- boundary tiles: combine the parked fragments in fixed (warp, slot) order and store
    __syncthreads();
    stamp(6);
    // slot tags in registers (lane q holds slot q): owner search and matching by ballot, and
    // the fragment loads issued together -- a serial walk over shared memory cost ~2 us here
    const int my_tag = lane < 2 * kWarps ? slot_tile[lane] : -1;
    for (int i = warp; i < 2 * kWarps; i += kWarps) {
      const int tile = __shfl_sync(0xffffffffu, my_tag, i);
      if (tile < 0) continue;
      const unsigned match = __ballot_sync(0xffffffffu, my_tag == tile);
      if (match & ((1u << i) - 1u)) continue;   // a lower slot holds this tile: it reduces
      float v[NT][4];
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) v[t][e] = 0.0f;
#pragma unroll
      for (int q = 0; q < 2 * kWarps; ++q) {   // fixed slot order: deterministic
        if (!((match >> q) & 1u)) continue;
        const float* src = red + q * kFrag;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) v[t][e] += src[(t * 4 + e) * 32 + lane];
      }
      store_tile(tile, v);
    }
    __syncthreads();   // slot_tile / red / csum / xs are reused by the next layer
  }
  stamp(5);
}

// ------------------------------------------------------------------------------------ host

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

size_t gemv_workspace_bytes(int, int, int) { return 0; }   // the GEMV needs no global workspace

constexpr size_t kXsBudget = 128 * 1024;  // stage activations in smem up to this size (if the whole plan fits)

template <int NT, int NW>
static int gemv_ns(int n_tiles, int nb, int grid) {
  using Cfg = GemvCfg<NT, NW>;
  const int tiles_max = (int)ceil_div(n_tiles, grid);
  const int ops = (int)ceil_div(ceil_div((int64_t)tiles_max * nb, Cfg::kWarps), Cfg::kSU);
  const int ns_max = kNSMax * 2 / Cfg::kSU;   // <= 8 units (8.4 KB) in flight per warp
  return ops >= ns_max ? ns_max : ops > 1 ? 2 : 1;
}

template <typename T, int NT, bool XS, int NW>
static int launch_gemv_x(const GemvArgs& a, int grid, int pdl, bool coop, cudaStream_t st) {
  auto kern = k_gemv_tq2<T, NT, XS, NW>;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured_dev = dev;
  }
  using Cfg = GemvCfg<NT, NW>;
  const int nrx = a.batch < 8 * NT ? a.batch : 8 * NT;
  const size_t smem = Cfg::smem(a.nb_max, nrx, XS, a.ns);
  if (smem > 227 * 1024) {
    set_error("tr_linear(gemv): %d blocks per row need %zu B of shared memory", a.nb_max, smem);
    return -1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(Cfg::kWarps * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (coop) {   // the persistent chain's grid barrier needs every CTA resident
    attrs[na].id = cudaLaunchAttributeCooperative;
    attrs[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) {
    set_error("tr_linear(gemv): launch failed: %s (grid %d, smem %zu)", cudaGetErrorString(e), grid, smem);
    return -1;
  }
  return 0;
}

template <int NT, int NW>
static bool xs_fits(int batch, int nb_max, int ns) {
  const int nrx = batch < 8 * NT ? batch : 8 * NT;
  return (size_t)nrx * GemvCfg<NT, NW>::x_stride(nb_max) <= kXsBudget &&
         GemvCfg<NT, NW>::smem(nb_max, nrx, true, ns) <= 227 * 1024;
}

template <typename T, int NT, int NW>
static int launch_gemv(GemvArgs& a, int grid, int pdl, bool coop, cudaStream_t st) {
  if (xs_fits<NT, NW>(a.batch, a.nb_max, a.ns)) return launch_gemv_x<T, NT, true, NW>(a, grid, pdl, coop, st);
  if (coop) {
    set_error("tr_linear_chain: activations of %d blocks x batch %d do not fit in shared memory", a.nb_max, a.batch);
    return -1;
  }
  return launch_gemv_x<T, NT, false, NW>(a, grid, pdl, coop, st);
}

// units per CTA at or below which the 8-warp, two-CTAs-per-SM variant wins (measured)
constexpr int kSmallCtaUnits = 48;
static bool small_variant(int n_tiles, int nb, int grid) { return (int64_t)ceil_div(n_tiles, grid) * nb <= kSmallCtaUnits; }

// true when the GEMV can stage this batch's activations in shared memory (its fast path)
bool gemv_stages_x(int batch, int rows, int cols) {
  if (batch > 8) return false;
  const int nb = (int)ceil_div(cols, kBlock), n_tiles = (int)ceil_div(rows, 16);
  const int grid = sm_count() < n_tiles ? sm_count() : n_tiles;
  if (small_variant(n_tiles, nb, grid)) return xs_fits<1, 8>(batch, nb, gemv_ns<1, 8>(n_tiles, nb, grid));
  return xs_fits<1, 16>(batch, nb, gemv_ns<1, 16>(n_tiles, nb, grid));
}

static GemvLayer make_layer(const void* w, const void* x, void* y, int64_t ldx, int64_t ldy, int rows, int cols) {
  GemvLayer L;
  L.w = (const uint8_t*)w;
  L.x = x;
  L.y = y;
  L.ldx = ldx;
  L.ldy = ldy;
  L.rows = rows;
  L.cols = cols;
  L.nb = (int)ceil_div(cols, kBlock);
  L.n_tiles = (int)ceil_div(rows, 16);
  L.x_vec = ((ldx % 8) == 0 && ((uintptr_t)x % 16) == 0) ? 1 : 0;
  L.pad_ = 0;
  return L;
}

int gemv_tq2(int act, const void* w, const void* x, void* y, int64_t ldx, int64_t ldy, int batch, int rows,
             int cols, int ctas, int pdl, cudaStream_t st, int pre, const void* pre_delta, const void* pre_gamma,
             void* pre_out, float eps, int out_f32) {
  GemvArgs a = {};
  a.out_f32 = out_f32;
  a.pre = pre;
  a.pre_delta = pre_delta;
  a.pre_gamma = pre_gamma;
  a.pre_out = pre_out;
  a.eps = eps;
  if (pre && (batch > 8 || !gemv_stages_x(batch, rows, cols))) {
    set_error("tr_linear_pre: fused producers need batch <= 8 and activations that fit in shared memory");
    return -1;
  }
  a.dbg = (ctas >> 12) & 0xF;
  ctas &= 0xFFF;
  a.l0 = make_layer(w, x, y, ldx, ldy, rows, cols);
  a.layers = nullptr;
  a.bar = nullptr;
  a.n_layers = 1;
  a.nb_max = a.l0.nb;
  a.batch = batch;
  int grid = ctas > 0 ? ctas : sm_count();
  if (grid > a.l0.n_tiles) grid = a.l0.n_tiles;
  const int nt = batch <= 8 ? 1 : (batch <= 16 ? 2 : 4);
  const bool small = small_variant(a.l0.n_tiles, a.l0.nb, grid);
  const bool bf = act != kActF16;
  if (nt == 1 && small) {
    a.ns = gemv_ns<1, 8>(a.l0.n_tiles, a.l0.nb, grid);
    return bf ? launch_gemv<__nv_bfloat16, 1, 8>(a, grid, pdl, false, st) : launch_gemv<__half, 1, 8>(a, grid, pdl, false, st);
  }
  if (nt == 1) {
    a.ns = gemv_ns<1, 16>(a.l0.n_tiles, a.l0.nb, grid);
    return bf ? launch_gemv<__nv_bfloat16, 1, 16>(a, grid, pdl, false, st)
              : launch_gemv<__half, 1, 16>(a, grid, pdl, false, st);
  }
  if (nt == 2) {
    a.ns = gemv_ns<2, 16>(a.l0.n_tiles, a.l0.nb, grid);
    return bf ? launch_gemv<__nv_bfloat16, 2, 16>(a, grid, pdl, false, st)
              : launch_gemv<__half, 2, 16>(a, grid, pdl, false, st);
  }
  a.ns = gemv_ns<4, 8>(a.l0.n_tiles, a.l0.nb, grid);
  return bf ? launch_gemv<__nv_bfloat16, 4, 8>(a, grid, pdl, false, st) : launch_gemv<__half, 4, 8>(a, grid, pdl, false, st);
}


}  // namespace tr
