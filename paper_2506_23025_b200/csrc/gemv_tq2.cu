// K3: decode-side ternary GEMV/skinny-GEMM, batch 1..32, TQ2 (2-bit) weights.
//
// Semantics (reference linear.py:1-13, _kernels.pyx:136-168; paper App. F):
//   y[n, r] = sum_b s[r, b] * (sum_{k in block b} trit[r, k] * x[n, k])
// with fp16/bf16 activations, the per-block inner sum accumulated in fp32 and
// the fp32 block partial scaled by the fp32 value of the binary16 scale, blocks
// accumulated in ascending order inside a K-split; splits are reduced in
// ascending order.  Output rounded once (RNE) to the activation dtype.
//
// B200 mapping: the kernel is HBM-bound at batch <= 16, so the
// instruction budget per weight is what matters (~1.4 lane-ops/weight at
// 6.5 TB/s).  Weights stream straight from HBM into registers with 128-bit
// ld.global.nc (the T16 layout makes every warp load 512 contiguous bytes),
// are expanded to fp16/bf16 trits with one LOP3 (mask | magic exponent) and one
// HFMA2 per two weights, and go directly into mma.sync.m16n8k16 A fragments:
// the tensor core does the +-x accumulation for up to 8 activation vectors
// per n8 tile at no extra ALU cost.  x for the CTA's K range is staged once in
// shared memory (padded, conflict-free LDS.128).  K is split across the CTAs of
// a thread-block cluster (<= 8) and reduced deterministically through DSMEM.
// Weight loads for the first stages are issued before griddepcontrol.wait so a
// PDL-chained layer overlaps its weight fetch with the previous kernel's tail.
#include <cooperative_groups.h>
#include "common.cuh"

namespace cg = cooperative_groups;

namespace tr {

constexpr int kGemvWarps = 4;
constexpr int kXChunkBytes = 144;               // 64 halves + 16 B pad (bank spread)
constexpr int kXBlockBytes = 4 * kXChunkBytes;  // one 256-block of one activation row

__host__ __device__ inline int x_row_stride(int kb) {
  int r = kb * kXBlockBytes;
  return (r % 128 == 64) ? r : r + 64;   // rows g, g+1 land in opposite bank halves
}

template <typename T> struct Frag;
template <> struct Frag<__half> {
  // 2-bit digit field j of each 16-bit half -> half2 trit in {-1,0,1}:
  // (w & (3<<2j)) | 0x6400 == 1024 + 4^j d ; * 4^-j - (1024*4^-j + 1) == d - 1 (exact).
  __device__ static void decode8(uint32_t w, uint32_t (&o)[8]) {
    const __half2 s0 = __float2half2_rn(1.0f), s1 = __float2half2_rn(0.25f), s2 = __float2half2_rn(0.0625f),
                  s3 = __float2half2_rn(0.015625f);
    const __half2 c0 = __float2half2_rn(-1025.0f), c1 = __float2half2_rn(-257.0f), c2 = __float2half2_rn(-65.0f),
                  c3 = __float2half2_rn(-17.0f);
    uint32_t hi = w >> 8;
    uint32_t v[8] = {lop3_and_or(w, 0x00030003u, 0x64006400u), lop3_and_or(w, 0x000C000Cu, 0x64006400u),
                     lop3_and_or(w, 0x00300030u, 0x64006400u), lop3_and_or(w, 0x00C000C0u, 0x64006400u),
                     lop3_and_or(hi, 0x00030003u, 0x64006400u), lop3_and_or(hi, 0x000C000Cu, 0x64006400u),
                     lop3_and_or(hi, 0x00300030u, 0x64006400u), lop3_and_or(hi, 0x00C000C0u, 0x64006400u)};
    const __half2 sc[4] = {s0, s1, s2, s3}, cc[4] = {c0, c1, c2, c3};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      __half2 r = __hfma2(*reinterpret_cast<__half2*>(&v[k]), sc[k & 3], cc[k & 3]);
      o[k] = *reinterpret_cast<uint32_t*>(&r);
    }
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
  // bf16 has 7 mantissa bits: magic 0x4300 (=128) holds fields at bits 0..5, so
  // fields at bits 6..7 / 14..15 are shifted down first.
  __device__ static void decode8(uint32_t w, uint32_t (&o)[8]) {
    const uint32_t M = 0x43004300u;
    uint32_t a6 = w >> 6, a8 = w >> 8, a14 = w >> 14;
    uint32_t v[8] = {lop3_and_or(w, 0x00030003u, M),  lop3_and_or(w, 0x000C000Cu, M),
                     lop3_and_or(w, 0x00300030u, M),  lop3_and_or(a6, 0x00030003u, M),
                     lop3_and_or(a8, 0x00030003u, M), lop3_and_or(a8, 0x000C000Cu, M),
                     lop3_and_or(a8, 0x00300030u, M), lop3_and_or(a14, 0x00030003u, M)};
    const float scf[8] = {1.0f, 0.25f, 0.0625f, 1.0f, 1.0f, 0.25f, 0.0625f, 1.0f};
    const float ccf[8] = {-129.0f, -33.0f, -9.0f, -129.0f, -129.0f, -33.0f, -9.0f, -129.0f};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      __nv_bfloat162 r = __hfma2(*reinterpret_cast<__nv_bfloat162*>(&v[k]), __float2bfloat162_rn(scf[k]),
                                 __float2bfloat162_rn(ccf[k]));
      o[k] = *reinterpret_cast<uint32_t*>(&r);
    }
  }
  __device__ static void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
};

struct GemvArgs {
  const uint4* w;        // T16 tile-blocks
  const uint32_t* sc;    // T16 half2 scale pairs
  const void* x;         // [batch][ldx] activations
  void* y;               // [batch][ldy] outputs
  int64_t ldx, ldy;
  int rows, cols, nb, n_tiles, batch, ks;
  int x_vec;             // 1 if 16-byte vector loads of x are legal
};

template <typename T, int NT, int S>
__global__ void __launch_bounds__(kGemvWarps * 32) k_gemv_tq2(GemvArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // [split-K partials (cluster-visible, same offset in every CTA)] [x slice]
  constexpr int kRedBytes = kGemvWarps * NT * 4 * 32 * 4;
  float* red = reinterpret_cast<float*>(smem_raw);
  uint8_t* smem = smem_raw + (a.ks > 1 ? kRedBytes : 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int tile = blockIdx.x * kGemvWarps + warp;
  const int sp = blockIdx.y;
  const int kb0 = (int)((int64_t)sp * a.nb / a.ks), kb1 = (int)((int64_t)(sp + 1) * a.nb / a.ks);
  const int KB = kb1 - kb0;
  const int xrs = x_row_stride(KB);
  const int nrows_x = a.batch < 8 * NT ? a.batch : 8 * NT;

  // ---- prologue: weight + scale loads for the first S blocks (independent of x)
  uint4 wl[S], wh[S];
  uint32_t sv[S];
#pragma unroll
  for (int st = 0; st < S; ++st) {
    if (st < KB) {
      const int64_t tb = (int64_t)(kb0 + st) * a.n_tiles + tile;
      wl[st] = ldg_nc_v4(a.w + tb * 64 + c * 8 + g);
      wh[st] = ldg_nc_v4(a.w + tb * 64 + 32 + c * 8 + g);
      sv[st] = ldg_nc_u32(a.sc + tb * 8 + g);
    }
  }
  griddep_launch_dependents();
  griddep_wait();   // x is produced by the previous kernel in the stream

  // ---- stage x[0:nrows_x, kb0*256 : kb1*256] into shared memory
  {
    const T* xg = reinterpret_cast<const T*>(a.x);
    const int64_t kbase = (int64_t)kb0 * kBlock;
    const int units = nrows_x * KB * 32;   // 16-byte units (8 elements)
    for (int u = threadIdx.x; u < units; u += blockDim.x) {
      const int n = u / (KB * 32), rem = u % (KB * 32);
      const int blk = rem >> 5, cu = rem & 31, ch = cu >> 3, q = cu & 7;
      const int64_t k = kbase + blk * kBlock + ch * 64 + q * 8;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (a.x_vec && k + 8 <= a.cols) {
        v = *reinterpret_cast<const uint4*>(xg + n * a.ldx + k);
      } else {
        T tmp[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) tmp[e] = (k + e < a.cols) ? xg[n * a.ldx + k + e] : Act<T>::from_float(0.0f);
        v = *reinterpret_cast<uint4*>(tmp);
      }
      *reinterpret_cast<uint4*>(smem + n * xrs + blk * kXBlockBytes + ch * kXChunkBytes + q * 16) = v;
    }
  }
  __syncthreads();

  float acc[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[t][e] = 0.0f;

  for (int base = 0; base < KB; base += S) {
#pragma unroll
    for (int st = 0; st < S; ++st) {
      const int kbi = base + st;
      if (kbi < KB) {
        float bacc[NT][4];
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) bacc[t][e] = 0.0f;
        const uint8_t* xb = smem + kbi * kXBlockBytes + c * kXChunkBytes;
        const uint32_t wlv[4] = {wl[st].x, wl[st].y, wl[st].z, wl[st].w};
        const uint32_t whv[4] = {wh[st].x, wh[st].y, wh[st].z, wh[st].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4 xv[NT][2];
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int n = 8 * t + g;
            if (n < nrows_x) {
              xv[t][0] = *reinterpret_cast<const uint4*>(xb + n * xrs + (2 * i) * 16);
              xv[t][1] = *reinterpret_cast<const uint4*>(xb + n * xrs + (2 * i + 1) * 16);
            } else {
              xv[t][0] = make_uint4(0, 0, 0, 0);
              xv[t][1] = make_uint4(0, 0, 0, 0);
            }
          }
          uint32_t lo[8], hi[8];
          Frag<T>::decode8(wlv[i], lo);
          Frag<T>::decode8(whv[i], hi);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const uint32_t A[4] = {lo[2 * qq], hi[2 * qq], lo[2 * qq + 1], hi[2 * qq + 1]};
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const uint4& u = xv[t][qq >> 1];
              const uint32_t b0 = (qq & 1) ? u.z : u.x, b1 = (qq & 1) ? u.w : u.y;
              Frag<T>::mma(bacc[t], A, b0, b1);
            }
          }
        }
        const __half2 sp2 = *reinterpret_cast<const __half2*>(&sv[st]);
        const float s_lo = __low2float(sp2), s_hi = __high2float(sp2);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          acc[t][0] = __fadd_rn(acc[t][0], __fmul_rn(s_lo, bacc[t][0]));
          acc[t][1] = __fadd_rn(acc[t][1], __fmul_rn(s_lo, bacc[t][1]));
          acc[t][2] = __fadd_rn(acc[t][2], __fmul_rn(s_hi, bacc[t][2]));
          acc[t][3] = __fadd_rn(acc[t][3], __fmul_rn(s_hi, bacc[t][3]));
        }
        // refill this stage with block kbi + S
        const int nk = kbi + S;
        if (nk < KB) {
          const int64_t tb = (int64_t)(kb0 + nk) * a.n_tiles + tile;
          wl[st] = ldg_nc_v4(a.w + tb * 64 + c * 8 + g);
          wh[st] = ldg_nc_v4(a.w + tb * 64 + 32 + c * 8 + g);
          sv[st] = ldg_nc_u32(a.sc + tb * 8 + g);
        }
      }
    }
  }

  T* y = reinterpret_cast<T*>(a.y);
  const int r0 = tile * 16 + g, r1 = r0 + 8;
  if (a.ks == 1) {
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int n0 = 8 * t + 2 * c, n1 = n0 + 1;
      if (n0 < a.batch) {
        if (r0 < a.rows) y[n0 * a.ldy + r0] = Act<T>::from_float(acc[t][0]);
        if (r1 < a.rows) y[n0 * a.ldy + r1] = Act<T>::from_float(acc[t][2]);
      }
      if (n1 < a.batch) {
        if (r0 < a.rows) y[n1 * a.ldy + r0] = Act<T>::from_float(acc[t][1]);
        if (r1 < a.rows) y[n1 * a.ldy + r1] = Act<T>::from_float(acc[t][3]);
      }
    }
    return;
  }

  // ---- split-K reduction across the cluster through distributed shared memory
  constexpr int kEntries = kGemvWarps * NT * 4 * 32;
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < 4; ++e) red[((warp * NT + t) * 4 + e) * 32 + lane] = acc[t][e];
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();
  const int ks = a.ks;
  const int e0 = sp * kEntries / ks, e1 = (sp + 1) * kEntries / ks;
  for (int idx = e0 + threadIdx.x; idx < e1; idx += blockDim.x) {
    const int ln = idx & 31, e = (idx >> 5) & 3, t = (idx >> 7) % NT, w = (idx >> 7) / NT;
    const int gg = ln >> 2, cc = ln & 3;
    const int row = (blockIdx.x * kGemvWarps + w) * 16 + gg + ((e & 2) ? 8 : 0);
    const int n = 8 * t + 2 * cc + (e & 1);
    if (n < a.batch && row < a.rows) {
      float v = 0.0f;
      for (int q = 0; q < ks; ++q) v = __fadd_rn(v, cluster.map_shared_rank(red, q)[idx]);
      y[n * a.ldy + row] = Act<T>::from_float(v);
    }
  }
  cluster.sync();
}

template <typename T, int NT, int S>
static int launch_gemv(const GemvArgs& a, int pdl, cudaStream_t st) {
  auto kern = k_gemv_tq2<T, NT, S>;
  const int nrows_x = a.batch < 8 * NT ? a.batch : 8 * NT;
  const int kbmax = (int)ceil_div(a.nb, a.ks);
  const size_t smem = (size_t)nrows_x * x_row_stride(kbmax) + (a.ks > 1 ? kGemvWarps * NT * 4 * 32 * 4 : 0);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.n_tiles / kGemvWarps, a.ks, 1);
  cfg.blockDim = dim3(kGemvWarps * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (a.ks > 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = 1;
    attrs[na].val.clusterDim.y = a.ks;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) {
    set_error("tr_linear(gemv): launch failed: %s", cudaGetErrorString(e));
    return -1;
  }
  return 0;
}

// Host-side split heuristic: fill the 148 SMs with ~4 resident CTAs each, keep
// the per-CTA x slice within the shared-memory budget.
int gemv_choose_ks(int n_tiles, int nb, int batch_rows) {
  const int row_ctas = n_tiles / kGemvWarps;
  int ks = (int)ceil_div(148 * 4, row_ctas);
  if (ks > 8) ks = 8;
  if (ks > nb) ks = nb;
  if (ks < 1) ks = 1;
  while (ks < 8 && ks < nb && (int64_t)batch_rows * x_row_stride((int)ceil_div(nb, ks)) > 160 * 1024) ++ks;
  return ks;
}

int gemv_tq2(int act, const void* w, const void* x, void* y, int64_t ldx, int64_t ldy, int batch, int rows,
             int cols, int ks, int pdl, cudaStream_t st) {
  GemvArgs a;
  const int nb = (int)ceil_div(cols, kBlock);
  const int n_tiles = (int)(rows_padded(rows) / 16);
  a.w = (const uint4*)w;
  a.sc = (const uint32_t*)((const uint8_t*)w + (int64_t)nb * n_tiles * kTileBlockBytes);
  a.x = x;
  a.y = y;
  a.ldx = ldx;
  a.ldy = ldy;
  a.rows = rows;
  a.cols = cols;
  a.nb = nb;
  a.n_tiles = n_tiles;
  a.batch = batch;
  const int nt = batch <= 8 ? 1 : (batch <= 16 ? 2 : 4);
  a.ks = ks > 0 ? ks : gemv_choose_ks(n_tiles, nb, batch < 8 * nt ? batch : 8 * nt);
  a.x_vec = ((ldx % 8) == 0 && ((uintptr_t)x % 16) == 0) ? 1 : 0;
  if (act == kActF16) {
    if (nt == 1) return launch_gemv<__half, 1, 4>(a, pdl, st);
    if (nt == 2) return launch_gemv<__half, 2, 4>(a, pdl, st);
    return launch_gemv<__half, 4, 3>(a, pdl, st);
  } else {
    if (nt == 1) return launch_gemv<__nv_bfloat16, 1, 4>(a, pdl, st);
    if (nt == 2) return launch_gemv<__nv_bfloat16, 2, 4>(a, pdl, st);
    return launch_gemv<__nv_bfloat16, 4, 3>(a, pdl, st);
  }
}

}  // namespace tr
