// K6: a chain of decode GEMVs (batch 1-4, TQ2) as ONE persistent launch.
//
// Each product is K3-S8's (gemv_s8.cu: activations on a per-block integer grid, int8 slices,
// u8 x s8 mma.sync, exact block sums; reference semantics linear.py:137-166).  What changes is
// the schedule.  A PDL chain of single-layer kernels pays, per layer, the launch release
// (1-1.5 us), the activation load and staging, and a main loop whose weights only started
// streaming when the kernel began -- ~6 us for a layer whose weights take 0.7-1.8 us to
// stream.  Here:
//  * one CTA per SM for the whole chain; every warp owns a TMA (cp.async.bulk) ring whose
//    producer walks the warp's weight units of op 0, then op 1, ... -- weights do not depend on
//    the activations, so the ring refills across op boundaries and HBM keeps streaming while
//    the grid waits for an op's inputs;
//  * op l's inputs are ready when every CTA has stored its part of op l-1: one release
//    (fence + atomicAdd) per CTA and op on a counter in the workspace, one acquiring poller
//    per CTA -- no kernel boundary, no CTA launch, no re-staging of weights;
//  * the fused producers of K3-S8 (add + RMSNorm, SiLU * up) and the SwiGLU epilogue are per-op
//    options, so a decoder layer's GEMVs chain without glue kernels;
//  * the counters are re-zeroed by the last CTA to finish, so the launch is replayable from a
//    CUDA graph with no host work.
// The kernel never triggers its dependents early (no griddepcontrol.launch_dependents): the
// next kernel starts after the last CTA exits, which also orders counter reuse.
#include <vector>

#include "s8_core.cuh"

namespace tr {

struct ChainOp {   // device table entry (host: from TrChainLayer)
  const uint8_t* w;
  const void* x;
  void* y;
  const void* delta;
  const void* gamma;
  void* x_out;
  int64_t ldx, ldy;
  int rows, cols, nb, n_tiles;
  int x_vec, pre, epi, out_f32;
  float eps;
  int pad_;
};

static_assert(sizeof(ChainOp) == 104, "graph.Chain.trace() mirrors the workspace layout");

struct ChainW {   // what a warp's weight producer needs per op (kept in shared memory)
  const uint8_t* w;
  int n_tiles_epi;   // n_tiles | epi << 30
  int nb;
};

struct ChainArgs {
  const ChainOp* ops;
  const ChainW* wtab;
  unsigned* done;    // [n_ops + 1] arrival counters; zero before a launch, re-zeroed by the last CTA
  uint64_t* trace;   // development probe: per (op, CTA) 4 %globaltimer stamps, or null
  int n_ops, batch, ns, nb_max, tv_floats;
};

constexpr int kChainWarps = 16;
constexpr int kChainMaxOps = 256;
constexpr int kChainCounterBytes = 4096;

struct ChainSmem {   // [mbarriers | slot tags | producer table | reduction | -Cs | grid factors | staged x | rings |
                     //  SwiGLU tiles]
  size_t tab, red, ncs, fsc, xs, ring, tv, total;
};
__host__ __device__ inline ChainSmem chain_smem(int ng, int nb_max, int nrx, int ns, int tv_floats, int n_ops) {
  ChainSmem m;
  m.tab = 1280;
  m.red = m.tab + (size_t)n_ops * sizeof(ChainW);
  m.ncs = m.red + (size_t)2 * kChainWarps * 64 * ng * 4;
  m.fsc = m.ncs + (size_t)nb_max * nrx * 16;
  m.xs = (m.fsc + (size_t)nb_max * nrx * 4 + 127) / 128 * 128;
  m.ring = m.xs + (size_t)nb_max * nrx * kS8ItemBytes;
  m.tv = m.ring + (size_t)kChainWarps * ns * kS8SU * kUnitBytes;
  m.total = m.tv + (size_t)tv_floats * 4;
  return m;
}

// The CTA's tiles [t0, t1) of an op (whole gate/up tile pairs with the SwiGLU epilogue) and
// warp w's contiguous unit range [u0, u1) of them -- K3-S8's ownership, per op.
__device__ __forceinline__ void chain_range(int n_tiles, int nb, int epi, int warp, unsigned& t0, unsigned& t1,
                                            int& u0, int& u1) {
  const unsigned tq = epi ? 2u : 1u, tn = (unsigned)n_tiles / tq;
  t0 = tq * (blockIdx.x * tn / gridDim.x);
  t1 = tq * ((blockIdx.x + 1) * tn / gridDim.x);
  const int LL = (int)(t1 - t0) * nb;
  u0 = (int)t0 * nb + (int)((unsigned)(warp * LL) / kChainWarps);
  u1 = (int)t0 * nb + (int)((unsigned)((warp + 1) * LL) / kChainWarps);
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Stage op o's activations (its fused producer first) as int8 slices: xs, -Cs, grid factors.
// Loads of data written inside this launch go through L2 (s8_load8_cg).
template <typename T>
__device__ void chain_stage(const ChainOp& o, int nbr, int nrx, int lr, uint8_t* xs, int32_t* ncs, float* fsc,
                            float* ss_buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = o.nb, n_items = nb * nrx;
  const T* xg = reinterpret_cast<const T*>(o.x);
  if (o.pre == TR_PRE_ADD_RMSNORM) {   // x = rmsnorm(x + delta) * gamma; CTA 0 stores x + delta
    const T* dg = reinterpret_cast<const T*>(o.delta);
    const T* gam = reinterpret_cast<const T*>(o.gamma);
    for (int item = warp; item < n_items; item += kChainWarps) {
      const int kb = item >> lr, br = item & (nrx - 1);
      const int64_t kx = (int64_t)kb * kBlock + lane * 8;
      const bool live = br < nbr;
      uint4 xv = make_uint4(0, 0, 0, 0), dv = make_uint4(0, 0, 0, 0);
      if (live) {
        xv = s8_load8_cg(xg + br * o.ldx, kx, o.cols, o.x_vec);
        if (dg) dv = s8_load8_cg(dg + br * o.ldx, kx, o.cols, o.x_vec);
      }
      float f[8];
      s8_f8<T>(xv, f);
      if (dg) {
        float d[8];
        s8_f8<T>(dv, d);
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = s8_rnd<T>(f[e] + d[e]);
      }
      const uint4 hv = s8_pack8<T>(f);
      *reinterpret_cast<uint4*>(xs + (size_t)item * kS8ItemBytes + lane * 16) = hv;   // parked in its own item
      if (blockIdx.x == 0 && o.x_out && kx < o.cols && live) {
        T* out = reinterpret_cast<T*>(o.x_out) + br * o.ldx + kx;
        if (kx + 8 <= o.cols && o.x_vec) {
          *reinterpret_cast<uint4*>(out) = hv;
        } else {
          const T* he = reinterpret_cast<const T*>(&hv);
          for (int e = 0; e < 8 && kx + e < o.cols; ++e) out[e] = he[e];
        }
      }
      float ss = 0.0f;
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += f[e] * f[e];
#pragma unroll
      for (int s = 16; s; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
      if (lane == 0) ss_buf[item] = ss;
    }
    __syncthreads();
    for (int item = warp; item < n_items; item += kChainWarps) {
      const int kb = item >> lr, br = item & (nrx - 1);
      const int64_t kx = (int64_t)kb * kBlock + lane * 8;
      float f[8], gm[8];
      s8_f8<T>(*reinterpret_cast<const uint4*>(xs + (size_t)item * kS8ItemBytes + lane * 16), f);
      s8_f8<T>(s8_load8(gam, kx, o.cols, o.x_vec), gm);
      float ss = 0.0f;   // the same fixed-order sum in every warp and CTA
      for (int q = lane; q < nb; q += 32) ss += ss_buf[q * nrx + br];
#pragma unroll
      for (int s = 16; s; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
      const float iv = rsqrtf(ss / o.cols + o.eps);
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = s8_rnd<T>(s8_rnd<T>(f[e] * iv) * gm[e]);
      __syncwarp();   // every lane holds its h before the item's bytes are overwritten
      s8_stage_block(f, xs, ncs, fsc, nrx, kb, br);
    }
    return;
  }
  // plain x, or silu(gate) * up of a gate|up product; loads for 4 items in flight
  for (int i0 = warp; i0 < n_items; i0 += 4 * kChainWarps) {
    uint4 va[4], vb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int item = i0 + i * kChainWarps;
      va[i] = vb[i] = make_uint4(0, 0, 0, 0);
      if (item < n_items) {
        const int kb = item >> lr, br = item & (nrx - 1);
        const int64_t kx = (int64_t)kb * kBlock + lane * 8;
        if (br < nbr) {
          va[i] = s8_load8_cg(xg + br * o.ldx, kx, o.cols, o.x_vec);
          if (o.pre == TR_PRE_SILU_MUL) vb[i] = s8_load8_cg(xg + br * o.ldx + o.cols, kx, o.cols, o.x_vec);
        }
      }
    }
#pragma unroll 1
    for (int i = 0; i < 4; i += 2) {
      float f[2][8];
      int kbs[2], brs[2];
      int nv = 0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int item = i0 + (i + t) * kChainWarps;
        const int it = item < n_items ? item : i0;
        kbs[t] = it >> lr;
        brs[t] = it & (nrx - 1);
        nv += item < n_items;
        s8_f8<T>(va[i + t], f[t]);
        if (o.pre == TR_PRE_SILU_MUL) {
          float up[8];
          s8_f8<T>(vb[i + t], up);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            f[t][e] = s8_rnd<T>(s8_rnd<T>(__fdividef(f[t][e], 1.0f + __expf(-f[t][e]))) * up[e]);
        }
      }
      if (nv > 0) s8_stage_blocks<2>(f, xs, ncs, fsc, nrx, kbs, brs, nv);
    }
  }
}

template <typename T, int NG>
__global__ void __launch_bounds__(kChainWarps * 32, 1) k_gemv_chain(const ChainArgs a) {
  constexpr int NW = kChainWarps;
  constexpr int kSlotBytes = kS8SU * kUnitBytes;
  extern __shared__ __align__(128) uint8_t smem[];
  const int NS = a.ns, nbr = a.batch;
  const int nrx = NG == 2 ? 4 : nbr, lr = NG == 2 ? 2 : nbr - 1;
  const ChainSmem L = chain_smem(NG, a.nb_max, nrx, NS, a.tv_floats, a.n_ops);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);   // NW * NS <= 128
  int* slot_tile = reinterpret_cast<int*>(smem + 1024);   // 2 * NW
  ChainW* wtab = reinterpret_cast<ChainW*>(smem + L.tab);
  for (int i = threadIdx.x; i < a.n_ops; i += blockDim.x) wtab[i] = a.wtab[i];
  __syncthreads();
  float* red = reinterpret_cast<float*>(smem + L.red);
  int32_t* ncs = reinterpret_cast<int32_t*>(smem + L.ncs);
  float* fsc = reinterpret_cast<float*>(smem + L.fsc);
  uint8_t* xs = smem + L.xs;
  uint8_t* ring = smem + L.ring;
  float* tv = reinterpret_cast<float*>(smem + L.tv);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const unsigned G = gridDim.x;
  uint64_t* mybar = bars + warp * NS;
  uint8_t* myring = ring + warp * NS * kSlotBytes;
  auto stamp = [&](int l, int k) {
    if (a.trace && threadIdx.x == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      a.trace[((size_t)l * G + blockIdx.x) * 4 + k] = t;
    }
  };

  // ---- weight producer (lane 0 of each warp): the warp's units of op 0, op 1, ... in order
  int pl = 0, pu = 0, pu1 = 0;
  const uint8_t* pw = nullptr;
  uint64_t pol = 0;
  auto producer_seek = [&]() {   // skip to the next op in which this warp owns units
    while (pu >= pu1 && ++pl < a.n_ops) {
      const ChainW o = wtab[pl];
      unsigned t0_, t1_;
      chain_range(o.n_tiles_epi & 0x3FFFFFFF, o.nb, o.n_tiles_epi >> 30, warp, t0_, t1_, pu, pu1);
      pw = o.w;
    }
  };
  auto issue = [&](int slot) {
    if (pl >= a.n_ops) return;
    const int n = min(kS8SU, pu1 - pu);
    mbar_expect_tx(&mybar[slot], n * kUnitBytes);
    bulk_g2s(myring + slot * kSlotBytes, pw + (int64_t)pu * kUnitBytes, n * kUnitBytes, &mybar[slot], pol);
    pu += n;
    if (pu >= pu1) producer_seek();
  };
  if (lane == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < NS; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
    const ChainW o0 = wtab[0];
    unsigned t0_, t1_;
    chain_range(o0.n_tiles_epi & 0x3FFFFFFF, o0.nb, o0.n_tiles_epi >> 30, warp, t0_, t1_, pu, pu1);
    pw = o0.w;
    if (pu >= pu1) producer_seek();
    for (int s = 0; s < NS; ++s) issue(s);   // weights do not depend on x: before the wait
  }
  __syncwarp();

  int slot = 0;           // consumer ring position (continues across ops)
  uint32_t phase = 0;
  int refill = -1;        // slot consumed last, refilled at the next iteration (its loads are done)
  const uint32_t xs_base = smem_u32(xs);
  const float lane_w = (c & 1) ? 65536.0f : 1.0f;

  for (int l = 0; l < a.n_ops; ++l) {
    const ChainOp o = a.ops[l];
    const int nb = o.nb;
    stamp(l, 0);
    if (l == 0) {
      griddep_wait();   // the first op's inputs belong to the previous kernel until here
    } else {
      if (threadIdx.x == 0)
        while (ld_acquire_gpu(a.done + (l - 1)) < G) {
        }
      __syncthreads();   // every CTA has stored op l-1 (and all earlier ops)
    }
    if (lane == 0) {
      slot_tile[2 * warp] = -1;
      slot_tile[2 * warp + 1] = -1;
    }
    stamp(l, 1);
    chain_stage<T>(o, nbr, nrx, lr, xs, ncs, fsc, red);
    __syncthreads();
    stamp(l, 2);

    unsigned t0, t1;
    int wu0, wu1;
    chain_range(o.n_tiles, nb, o.epi, warp, t0, t1, wu0, wu1);
    uint32_t xsB32[NG];
    const int32_t* ncsD[NG];
    const float* fscD[NG];
#pragma unroll
    for (int G2 = 0; G2 < NG; ++G2) {
      const int nBc = NG == 1 ? (g & (4 * nrx - 1)) : 8 * G2 + g;
      const int bB = nBc >> 2, sB = nBc & 3;
      const int swB = ((c >> 1) << 1) | (sB & 1);
      xsB32[G2] = (xs_base + (uint32_t)(bB * kS8ItemBytes + sB * 256 + c * 64)) ^ (uint32_t)(swB << 4);
      const int bD = NG == 1 ? min(c >> 1, nrx - 1) : 2 * G2 + (c >> 1);
      ncsD[G2] = ncs + bD * 4 + 2 * (c & 1);
      fscD[G2] = fsc + bD;
    }
    const int kb_shift = 10 + lr;

    auto store_tile = [&](int tile, const float (&v)[NG][2]) {
      if (o.epi) {   // keep: the pair's other tile may come from another warp
#pragma unroll
        for (int G2 = 0; G2 < NG; ++G2) {
          const int row = 2 * G2 + (c >> 1);
          if ((c & 1) == 0 && row < nbr) {
            float* tt = tv + (size_t)(tile - (int)t0) * 64;
            tt[g * 4 + row] = v[G2][0];
            tt[(g + 8) * 4 + row] = v[G2][1];
          }
        }
        return;
      }
#pragma unroll
      for (int G2 = 0; G2 < NG; ++G2) {
        const int row = 2 * G2 + (c >> 1);
        if ((c & 1) == 0 && row < nbr) {
          const int r0 = tile * 16 + g, r1 = r0 + 8;
          if (r0 < o.rows) store_y<T>(o.y, (int64_t)row * o.ldy + r0, v[G2][0], o.out_f32);
          if (r1 < o.rows) store_y<T>(o.y, (int64_t)row * o.ldy + r1, v[G2][1], o.out_f32);
        }
      }
    };
    const int first_tile = wu0 < wu1 ? wu0 / nb : -1;
    int cur = first_tile;
    float acc[NG][2];
#pragma unroll
    for (int G2 = 0; G2 < NG; ++G2) acc[G2][0] = acc[G2][1] = 0.0f;
    auto close_tile = [&](int tile) {
      float v[NG][2];
#pragma unroll
      for (int G2 = 0; G2 < NG; ++G2)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          v[G2][e] = acc[G2][e] * lane_w;
          v[G2][e] += __shfl_xor_sync(0xffffffffu, v[G2][e], 1);
        }
      if (tile * nb >= wu0 && (tile + 1) * nb <= wu1) {
        store_tile(tile, v);
        return;
      }
      const int which = (tile == first_tile) ? 0 : 1;
      float* dst = red + (2 * warp + which) * 64 * NG;
#pragma unroll
      for (int G2 = 0; G2 < NG; ++G2) {
        dst[G2 * 64 + lane] = v[G2][0];
        dst[G2 * 64 + 32 + lane] = v[G2][1];
      }
      if (lane == 0) slot_tile[2 * warp + which] = tile;
    };
    auto mma_unit = [&](const uint4& wl, const uint4& wh, int kbq, int (&D)[NG][4]) {
      uint4 xw[NG][4];
      int2 cs[NG];
#pragma unroll
      for (int G2 = 0; G2 < NG; ++G2) {
        const uint32_t xp = xsB32[G2] + ((uint32_t)kbq << kb_shift);
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) xw[G2][i4] = ld_shared_v4u(xp ^ (i4 << 4));
        cs[G2] = *reinterpret_cast<const int2*>(ncsD[G2] + (kbq << (lr + 2)));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int w = i >> 1, j0 = 2 * (i & 1);
        const uint32_t m0 = 0x03030303u << (2 * j0), m1 = 0x03030303u << (2 * j0 + 2);
        const uint32_t lw = u4c(wl, w), hw = u4c(wh, w);
        const uint32_t A[4] = {lw & m0, hw & m0, lw & m1, hw & m1};
#pragma unroll
        for (int G2 = 0; G2 < NG; ++G2) {
          const uint32_t b0 = u4c(xw[G2][w], j0), b1 = u4c(xw[G2][w], j0 + 1);
          if (i == 0)
            imma_c(D[G2], A, b0, b1, cs[G2].x, cs[G2].y, cs[G2].x, cs[G2].y);
          else
            imma(D[G2], A, b0, b1);
        }
      }
    };
    auto epilogue = [&](const int (&d)[NG][4], uint32_t sv, int kbq) {
      const float2 sc = __half22float2(*reinterpret_cast<const __half2*>(&sv));
#pragma unroll
      for (int G2 = 0; G2 < NG; ++G2) {
        const float fb = fscD[G2][kbq * nrx];
        const int v0 = d[G2][0] + d[G2][1] * 256, v1 = d[G2][2] + d[G2][3] * 256;
        acc[G2][0] = fmaf((float)v0, sc.x * fb, acc[G2][0]);
        acc[G2][1] = fmaf((float)v1, sc.y * fb, acc[G2][1]);
      }
    };

    int kb = wu0 < wu1 ? wu0 - first_tile * nb : 0;
#pragma unroll 1
    for (int u = wu0; u < wu1;) {
      if (refill >= 0) {   // the slot read last iteration: its loads completed (values were used)
        __syncwarp();
        if (lane == 0) {
          fence_proxy_async_smem();
          issue(refill);
        }
      }
      const int n = min(kS8SU, wu1 - u);
      mbar_wait(&mybar[slot], phase);
      const uint8_t* sp = myring + slot * kSlotBytes;
      uint4 wl[kS8SU], wh[kS8SU];
      uint32_t sv[kS8SU];
#pragma unroll
      for (int q = 0; q < kS8SU; ++q) {
        if (q < n) {
          wl[q] = lds128(sp + q * kUnitBytes + t16_word(0, c, g) * 16);
          wh[q] = lds128(sp + q * kUnitBytes + t16_word(1, c, g) * 16);
          sv[q] = *reinterpret_cast<const uint32_t*>(sp + q * kUnitBytes + kTileBlockBytes + g * 4);
        }
      }
      refill = slot;
      if (++slot == NS) {
        slot = 0;
        phase ^= 1u;
      }
      if (n == kS8SU && kb + kS8SU <= nb) {   // common case: both units inside the current tile --
        int D0[NG][4], D1[NG][4];             // two independent IMMA chains the scheduler interleaves
        mma_unit(wl[0], wh[0], kb, D0);
        mma_unit(wl[1], wh[1], kb + 1, D1);
        epilogue(D0, sv[0], kb);
        epilogue(D1, sv[1], kb + 1);
        kb += kS8SU;
        u += n;
        continue;
      }
#pragma unroll
      for (int q = 0; q < kS8SU; ++q) {
        if (q < n) {
          if (kb == nb) {   // next tile
            close_tile(cur);
#pragma unroll
            for (int G2 = 0; G2 < NG; ++G2) acc[G2][0] = acc[G2][1] = 0.0f;
            ++cur;
            kb = 0;
          }
          int D[NG][4];
          mma_unit(wl[q], wh[q], kb, D);
          epilogue(D, sv[q], kb);
          ++kb;
        }
      }
      u += n;
    }
    if (refill >= 0) {   // hand the last slot back now, not after the next op's input wait
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async_smem();
        issue(refill);
      }
      refill = -1;
    }
    if (cur >= 0) close_tile(cur);

    // ---- boundary tiles: combine the parked fragments in fixed (warp, slot) order and store
    __syncthreads();
    const int my_tag = lane < 2 * NW ? slot_tile[lane] : -1;
    for (int i = warp; i < 2 * NW; i += NW) {
      const int tile = __shfl_sync(0xffffffffu, my_tag, i);
      if (tile < 0) continue;
      const unsigned match = __ballot_sync(0xffffffffu, my_tag == tile);
      if (match & ((1u << i) - 1u)) continue;
      float v[NG][2];
#pragma unroll
      for (int G2 = 0; G2 < NG; ++G2) v[G2][0] = v[G2][1] = 0.0f;
      for (unsigned mq = match; mq; mq &= mq - 1) {
        const int q = __ffs(mq) - 1;
#pragma unroll
        for (int G2 = 0; G2 < NG; ++G2) {
          v[G2][0] += red[q * 64 * NG + G2 * 64 + lane];
          v[G2][1] += red[q * 64 * NG + G2 * 64 + 32 + lane];
        }
      }
      store_tile(tile, v);
    }
    if (o.epi) {   // silu(gate) * up with the roundings of the unfused gate|up store + tr_silu_mul
      __syncthreads();
      T* y = reinterpret_cast<T*>(o.y);
      const int npairs = (int)(t1 - t0) / 2, rows_out = o.rows / 2;
      for (int idx = threadIdx.x; idx < npairs * 16 * nbr; idx += NW * 32) {
        const int p = idx / (16 * nbr), r = (idx / nbr) % 16, br = idx % nbr;
        const float gt = s8_rnd<T>(tv[(size_t)(2 * p) * 64 + r * 4 + br]);
        const float up = s8_rnd<T>(tv[(size_t)(2 * p + 1) * 64 + r * 4 + br]);
        const int orow = ((int)t0 / 2 + p) * 16 + r;
        if (orow < rows_out) y[br * o.ldy + orow] = Act<T>::from_float(s8_rnd<T>(__fdividef(gt, 1.0f + __expf(-gt))) * up);
      }
    }
    __syncthreads();   // all of this CTA's outputs of op l are stored
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(a.done + l, 1u);
    }
    stamp(l, 3);
  }
  // the last CTA through re-zeroes the counters (every CTA has finished all its waits)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.done + a.n_ops, 1u) == G - 1) {
      for (int l = 0; l <= a.n_ops; ++l) a.done[l] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------------------------ host

static ChainOp make_op(const TrChainLayer& h) {
  ChainOp o = {};
  o.w = (const uint8_t*)h.w;
  o.x = h.x;
  o.y = h.y;
  o.delta = h.delta;
  o.gamma = h.gamma;
  o.x_out = h.x_out;
  o.ldx = h.ldx;
  o.ldy = h.ldy;
  o.rows = (int)h.rows;
  o.cols = (int)h.cols;
  o.nb = (int)ceil_div(h.cols, kBlock);
  o.n_tiles = (int)ceil_div(h.rows, 16);
  o.x_vec = ((h.ldx % 8) == 0 && ((uintptr_t)h.x % 16) == 0 &&
             (h.pre_op != TR_PRE_ADD_RMSNORM || !h.delta || ((uintptr_t)h.delta % 16) == 0) &&
             (h.pre_op != TR_PRE_ADD_RMSNORM || ((uintptr_t)h.gamma % 16) == 0) &&
             (h.pre_op != TR_PRE_ADD_RMSNORM || !h.x_out || ((uintptr_t)h.x_out % 16) == 0) &&
             (h.pre_op != TR_PRE_SILU_MUL || (h.cols % 8) == 0))
                ? 1
                : 0;
  o.pre = h.pre_op;
  o.epi = (h.flags & TR_LINEAR_EPI_SWIGLU) ? 1 : 0;
  o.out_f32 = (h.flags & TR_LINEAR_OUT_F32) ? 1 : 0;
  o.eps = h.eps;
  return o;
}

struct ChainPlan {
  int nb_max, ns, tv_floats, ng, nrx;
  size_t smem;
};

static int chain_plan(const std::vector<ChainOp>& ops, int batch, int grid, ChainPlan& p) {
  p.nb_max = 0;
  p.tv_floats = 0;
  for (const ChainOp& o : ops) {
    p.nb_max = o.nb > p.nb_max ? o.nb : p.nb_max;
    if (o.epi) {
      const int tv = (int)(2 * ceil_div(o.n_tiles / 2, grid) * 64);
      p.tv_floats = tv > p.tv_floats ? tv : p.tv_floats;
    }
  }
  p.ng = batch <= 2 ? 1 : 2;
  p.nrx = batch <= 2 ? batch : 4;
  const size_t cap = 227 * 1024;
  p.ns = 0;
  for (int ns = 8; ns >= 2; --ns) {
    const ChainSmem m = chain_smem(p.ng, p.nb_max, p.nrx, ns, p.tv_floats, (int)ops.size());
    if (m.total <= cap) {
      p.ns = ns;
      p.smem = m.total;
      break;
    }
  }
  if (p.ns == 0) {
    set_error("tr_linear_chain: activations of %d blocks x batch %d leave no room for the weight rings", p.nb_max,
              batch);
    return -1;
  }
  return 0;
}

// workspace: [counters 4 KiB | ChainOp table | ChainW table | trace (dev probe)]
static size_t chain_trace_off(int n_ops) {
  return ((size_t)kChainCounterBytes + (sizeof(ChainOp) + sizeof(ChainW)) * (size_t)n_ops + 255) / 256 * 256;
}
size_t chain_workspace_bytes(int n_ops) { return chain_trace_off(n_ops) + (size_t)n_ops * sm_count() * 4 * 8; }

static int check_ops(const TrChainLayer* h, int n, int batch) {
  TR_REQUIRE(n >= 1 && n <= kChainMaxOps, "tr_linear_chain: 1 <= n_layers <= %d", kChainMaxOps);
  TR_REQUIRE(batch >= 1 && batch <= 4, "tr_linear_chain: batch must be 1..4 (int8-slice GEMV)");
  for (int l = 0; l < n; ++l) {
    const TrChainLayer& L = h[l];
    TR_REQUIRE(L.rows >= 1 && L.cols >= 1 && L.rows < (1LL << 30) && L.cols < (1LL << 24),
               "tr_linear_chain: layer %d: bad shape %lld x %lld", l, (long long)L.rows, (long long)L.cols);
    TR_REQUIRE(((uintptr_t)L.w & 15) == 0, "tr_linear_chain: layer %d: weights must be 16-byte aligned", l);
    TR_REQUIRE(L.pre_op == 0 || L.pre_op == TR_PRE_ADD_RMSNORM || L.pre_op == TR_PRE_SILU_MUL,
               "tr_linear_chain: layer %d: bad pre_op %d", l, L.pre_op);
    TR_REQUIRE(L.pre_op != TR_PRE_ADD_RMSNORM || L.gamma != nullptr, "tr_linear_chain: layer %d: RMSNorm needs gamma",
               l);
    const bool epi = (L.flags & TR_LINEAR_EPI_SWIGLU) != 0;
    TR_REQUIRE(!epi || (L.rows % 32) == 0, "tr_linear_chain: layer %d: SwiGLU rows must be whole tile pairs", l);
    TR_REQUIRE(!(epi && (L.flags & TR_LINEAR_OUT_F32)), "tr_linear_chain: layer %d: OUT_F32 with SwiGLU", l);
    TR_REQUIRE(L.ldx >= (L.pre_op == TR_PRE_SILU_MUL ? 2 * L.cols : L.cols) && L.ldy >= (epi ? L.rows / 2 : L.rows),
               "tr_linear_chain: layer %d: leading dimensions", l);
  }
  return 0;
}

int gemv_chain_s8(int act, const TrChainLayer* host, int n, int batch, void* ws, size_t ws_bytes, int flags,
                  cudaStream_t st, bool upload) {
  if (check_ops(host, n, batch)) return -1;
  TR_REQUIRE(ws != nullptr && ws_bytes >= chain_workspace_bytes(n),
             "tr_linear_chain: workspace too small; size it with tr_linear_chain_workspace_size");
  std::vector<ChainOp> ops((size_t)n);
  for (int l = 0; l < n; ++l) ops[l] = make_op(host[l]);
  const int grid = sm_count();
  ChainPlan p;
  if (chain_plan(ops, batch, grid, p)) return -1;
  uint8_t* base = (uint8_t*)ws;
  ChainOp* dev_ops = (ChainOp*)(base + kChainCounterBytes);
  ChainW* dev_w = (ChainW*)(dev_ops + n);
  if (upload) {   // synchronous, outside any stream capture (tr_linear_chain_prepare)
    std::vector<ChainW> wt((size_t)n);
    for (int l = 0; l < n; ++l) wt[l] = ChainW{ops[l].w, ops[l].n_tiles | (ops[l].epi << 30), ops[l].nb};
    cudaError_t e = cudaMemcpy(dev_ops, ops.data(), sizeof(ChainOp) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dev_w, wt.data(), sizeof(ChainW) * n, cudaMemcpyHostToDevice);
    TR_REQUIRE(e == cudaSuccess, "tr_linear_chain_prepare: table upload failed: %s", cudaGetErrorString(e));
    return 0;
  }
  ChainArgs a = {};
  a.ops = dev_ops;
  a.wtab = dev_w;
  a.done = (unsigned*)base;
  a.trace = ((flags >> 24) & 2) ? (uint64_t*)(base + chain_trace_off(n)) : nullptr;
  a.n_ops = n;
  a.batch = batch;
  a.ns = p.ns;
  a.nb_max = p.nb_max;
  a.tv_floats = p.tv_floats;
  void (*kern)(const ChainArgs);
  if (act == kActF16)
    kern = p.ng == 1 ? k_gemv_chain<__half, 1> : k_gemv_chain<__half, 2>;
  else
    kern = p.ng == 1 ? k_gemv_chain<__nv_bfloat16, 1> : k_gemv_chain<__nv_bfloat16, 2>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kChainWarps * 32, 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  attrs[na].id = cudaLaunchAttributeCooperative;   // the op counters need every CTA resident
  attrs[na].val.cooperative = 1;
  ++na;
  if (flags & TR_LINEAR_PDL) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  TR_REQUIRE(e == cudaSuccess, "tr_linear_chain: launch failed: %s (grid %d, smem %zu)", cudaGetErrorString(e), grid,
             p.smem);
  return 0;
}

}  // namespace tr
