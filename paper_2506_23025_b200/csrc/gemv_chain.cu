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
#include <algorithm>
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
  uint64_t* trace;   // development probe: per (op, CTA) 8 %globaltimer stamps, or null
  int n_ops, batch, nb_max, tv_floats;
  size_t ring_bytes;
  int piece;         // bytes per bulk copy (an op slice is cut into pieces)
  int probe;         // development probes: 4 = skip the staging arithmetic, 8 = skip the MMAs
};

constexpr int kChainWarps = 15;   // consumer (math) warps; + 1 producer warp = 16: 4 warps per SM sub-partition, 128 registers each
constexpr int kChainMaxOps = 256;
constexpr int kChainCounterBytes = 4096;

constexpr int kChainBars = 4;
constexpr int kChainPiece = 16 * 1024;   // op barriers: ops l, l+1, .. l+3 may be in flight in the ring

struct ChainSmem {   // [op mbarriers | slot tags | op table | CTA tile ranges | op ring bases | reduction | -Cs |
                     //  grid factors | staged x | weight ring | SwiGLU tiles]
  size_t tab, rng, red, ncs, fsc, xs, ring, tv, total;
  size_t ring_bytes;
};
__host__ __device__ inline ChainSmem chain_smem(int ng, int nb_max, int nrx, size_t ring_bytes, int tv_floats,
                                                int n_ops) {
  ChainSmem m;
  m.tab = 1280;
  m.rng = m.tab + (size_t)n_ops * sizeof(ChainW);
  m.red = (m.rng + (size_t)n_ops * 8 + 15) / 16 * 16;
  m.ncs = m.red + (size_t)2 * kChainWarps * 64 * ng * 4;
  m.fsc = m.ncs + (size_t)nb_max * nrx * 16;
  m.xs = (m.fsc + (size_t)nb_max * nrx * 4 + 127) / 128 * 128;
  m.ring = m.xs + (size_t)nb_max * nrx * kS8ItemBytes;
  m.ring_bytes = ring_bytes;
  m.tv = m.ring + ring_bytes;
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

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

// the 16 consumer warps synchronise on named barrier 1 (the producer warp never joins)
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(kChainWarps * 32) : "memory");
}

__device__ __forceinline__ void cta_tiles(int n_tiles, int epi, unsigned& t0, unsigned& t1) {
  const unsigned tq = epi ? 2u : 1u, tn = (unsigned)n_tiles / tq;
  t0 = tq * (blockIdx.x * tn / gridDim.x);
  t1 = tq * ((blockIdx.x + 1) * tn / gridDim.x);
}

__device__ __forceinline__ void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Stage op o's activations (its fused producer first) as int8 slices: xs, -Cs, grid factors.
// Loads of data written inside this launch go through L2 (s8_load8_cg).
template <typename T>
__device__ __forceinline__ void chain_stage(const ChainOp& o, int nbr, int nrx, int lr, uint8_t* xs, int32_t* ncs, float* fsc,
                            float* ss_buf, uint64_t* tr) {
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
    consumers_sync();
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
#pragma unroll
    for (int i = 0; i < 4; i += 2) {   // (unrolled: va / vb stay in registers)
      if (i0 + i * kChainWarps >= n_items) break;
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
        if (tr && i == 0 && t == 0 && threadIdx.x == 0) {   // (dev probe: the first loads have landed)
          uint64_t ts;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ts) : "r"(__float_as_uint(f[0][0])));
          tr[6] = ts;
        }
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
__global__ void __launch_bounds__((kChainWarps + 1) * 32, 1) k_gemv_chain(const ChainArgs a) {
  constexpr int NW = kChainWarps;
  extern __shared__ __align__(128) uint8_t smem[];
  const int nbr = a.batch;
  const int nrx = NG == 2 ? 4 : nbr, lr = NG == 2 ? 2 : nbr - 1;
  const ChainSmem L = chain_smem(NG, a.nb_max, nrx, a.ring_bytes, a.tv_floats, a.n_ops);
  uint64_t* obar = reinterpret_cast<uint64_t*>(smem);            // kChainBars "op slice landed" barriers
  uint64_t* ebar = obar + kChainBars;                            // kChainBars "op slice consumed" barriers
  int* ring_base = reinterpret_cast<int*>(smem + 256);           // kChainBars op offsets in the ring
  ChainOp* opwin = reinterpret_cast<ChainOp*>(smem + 512);       // kChainBars op descriptors (416 B)
  int* slot_tile = reinterpret_cast<int*>(smem + 1024);          // 2 * NW
  ChainW* wtab = reinterpret_cast<ChainW*>(smem + L.tab);
  uint2* rng = reinterpret_cast<uint2*>(smem + L.rng);           // this CTA's tiles [t0, t1) per op
  float* red = reinterpret_cast<float*>(smem + L.red);
  int32_t* ncs = reinterpret_cast<int32_t*>(smem + L.ncs);
  float* fsc = reinterpret_cast<float*>(smem + L.fsc);
  uint8_t* xs = smem + L.xs;
  uint8_t* ring = smem + L.ring;
  float* tv = reinterpret_cast<float*>(smem + L.tv);
  const int R = (int)a.ring_bytes;   // a multiple of kUnitBytes: a unit never straddles the wrap
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const unsigned G = gridDim.x;
  auto stamp = [&](int l, int k) {   // (thread 0)
    if (a.trace && threadIdx.x == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      a.trace[((size_t)l * G + blockIdx.x) * 16 + k] = t;
    }
  };
  for (int i = threadIdx.x; i < a.n_ops; i += blockDim.x) {
    const ChainW w = a.wtab[i];
    wtab[i] = w;
    unsigned t0, t1;
    cta_tiles(w.n_tiles_epi & 0x3FFFFFFF, w.n_tiles_epi >> 30, t0, t1);
    rng[i] = make_uint2(t0, t1);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kChainBars; ++i) {
      mbar_init(&obar[i], 1);
      mbar_init(&ebar[i], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // ---- weight producer (warp kChainWarps, one lane): op l's CTA slice -- tiles [t0, t1) x all
  // blocks, ONE contiguous run of the tile-major layout -- as a few large bulk copies (split at
  // the ring's wrap) into a CTA ring, op after op, as soon as the consumers release ring space.
  // It never joins the consumers' barriers, so TMA back-pressure never stalls the math warps.
  auto op_bytes = [&](int l) {
    const uint2 t = rng[l];
    return (int)(t.y - t.x) * wtab[l].nb * kUnitBytes;
  };
  if (warp == kChainWarps) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int head = 0, used = 0, freed = 0;
      for (int l = 0; l < a.n_ops; ++l) {
        const int S = op_bytes(l);
        while (used + S > R || l - freed >= kChainBars) {   // wait for the oldest slice to be consumed
          // (polls with back-off: a spinning warp would take issue slots from the math warps of its
          // sub-partition, and those would then reach every CTA barrier last)
          while (!mbar_test(&ebar[freed % kChainBars], (uint32_t)(freed / kChainBars) & 1u)) __nanosleep(200);
          used -= op_bytes(freed);
          ++freed;
        }
        fence_proxy_async_smem();   // (the consumers' reads of the reused bytes precede the copies)
        uint64_t* bar = &obar[l % kChainBars];
        ring_base[l % kChainBars] = head;
        opwin[l % kChainBars] = a.ops[l];   // the descriptor rides on the same barrier as the weights
        if (a.trace) {   // stamp 7: op l's slice issued
          uint64_t t;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
          a.trace[((size_t)l * G + blockIdx.x) * 16 + 7] = t;
        }
        if (S == 0 || a.piece == 255 * 1024) {   // (dev knob piece 255: no weight traffic at all)
          mbar_arrive(bar);
        } else {
          mbar_expect_tx(bar, (uint32_t)S);
          const uint8_t* src = wtab[l].w + (size_t)rng[l].x * wtab[l].nb * kUnitBytes;
          int left = S, h = head;
          while (left > 0) {
            const int n = min(min(left, R - h), a.piece);
            bulk_g2s(ring + h, src, (uint32_t)n, bar, pol);
            src += n;
            left -= n;
            h += n;
            if (h == R) h = 0;
          }
        }
        head += S;
        if (head >= R) head -= R;
        used += S;
      }
    }
    return;   // (the producer warp exits; in-flight copies complete on the consumers' barriers)
  }

  const uint32_t xs_base = smem_u32(xs);
  const float lane_w = (c & 1) ? 65536.0f : 1.0f;

  for (int l = 0; l < a.n_ops; ++l) {
    stamp(l, 0);
    // op l's descriptor and weight slice (issued by the producer warp well ahead)
    mbar_wait(&obar[l % kChainBars], (uint32_t)(l / kChainBars) & 1u);
    const ChainOp o = opwin[l % kChainBars];
    const int nb = o.nb;
    if (l == 0) {
      griddep_wait();   // the first op's inputs belong to the previous kernel until here
    } else {
      if (threadIdx.x == 0 && !(a.probe & 1))   // (dev probe 1: no inter-CTA wait)
        while (ld_acquire_gpu(a.done + (l - 1)) < G) {
        }
      consumers_sync();   // every CTA has stored op l-1 (and all earlier ops)
    }
    if (lane == 0) {
      slot_tile[2 * warp] = -1;
      slot_tile[2 * warp + 1] = -1;
    }
    stamp(l, 1);
    if (!(a.probe & 4))
      chain_stage<T>(o, nbr, nrx, lr, xs, ncs, fsc, red,
                     a.trace ? a.trace + ((size_t)l * G + blockIdx.x) * 16 : nullptr);
    consumers_sync();
    stamp(l, 2);

    const uint2 tt = rng[l];
    const unsigned t0 = tt.x, t1 = tt.y;
    const int LL = (int)(t1 - t0) * nb;
    const int wu0 = (int)t0 * nb + (int)((unsigned)(warp * LL) / NW);
    const int wu1 = (int)t0 * nb + (int)((unsigned)((warp + 1) * LL) / NW);
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
            float* tp = tv + (size_t)(tile - (int)t0) * 64;
            tp[g * 4 + row] = v[G2][0];
            tp[(g + 8) * 4 + row] = v[G2][1];
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

    if (warp == 0) stamp(l, 5);
    // unit u sits at ring offset base + (u - t0 nb) * 1056 (mod R)
    int off = ring_base[l % kChainBars] + (wu0 - (int)t0 * nb) * kUnitBytes;
    if (off >= R) off -= R;
    const uint32_t wofs0 = t16_word(0, c, g) * 16, wofs1 = t16_word(1, c, g) * 16;
    int kb = wu0 < wu1 ? wu0 - first_tile * nb : 0;
#pragma unroll 1
    for (int u = wu0; u < wu1;) {
      const int n = min(kS8SU, wu1 - u);
      uint4 wl[kS8SU], wh[kS8SU];
      uint32_t sv[kS8SU];
#pragma unroll
      for (int q = 0; q < kS8SU; ++q) {
        if (q < n) {
          const uint8_t* up = ring + off;
          wl[q] = lds128(up + wofs0);
          wh[q] = lds128(up + wofs1);
          sv[q] = *reinterpret_cast<const uint32_t*>(up + kTileBlockBytes + g * 4);
          off += kUnitBytes;
          if (off == R) off = 0;
        }
      }
      if (a.probe & 8) {   // (dev probe: weights read, no arithmetic)
        kb += n;
        while (kb >= nb) {
          kb -= nb;
          ++cur;
        }
        u += n;
        continue;
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
    if (warp == 0) stamp(l, 4);
    if (cur >= 0) close_tile(cur);

    // ---- boundary tiles: combine the parked fragments in fixed (warp, slot) order and store
    consumers_sync();
    stamp(l, 8);
    if (threadIdx.x == 0) mbar_arrive(&ebar[l % kChainBars]);   // every warp is done with op l's slice
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
      consumers_sync();
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
    stamp(l, 9);
    consumers_sync();   // all of this CTA's outputs of op l are stored
    stamp(l, 10);
    if (threadIdx.x == 0) red_release_gpu_add(a.done + l, 1u);   // (release: the CTA's stores first)
    stamp(l, 3);
  }
  // the last CTA through re-zeroes the counters (every CTA has finished all its waits, and every
  // warp of this CTA has made its last release: the sync below)
  consumers_sync();
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
  int nb_max, tv_floats, ng, nrx;
  size_t ring_bytes, smem;
};

// the weight ring gets all shared memory the staged activations leave, in whole units; it must
// hold the largest per-CTA op slice (an op is one bulk transfer) -- ideally two or more
static int chain_plan(const std::vector<ChainOp>& ops, int batch, int grid, ChainPlan& p, size_t ring_cap) {
  p.nb_max = 0;
  p.tv_floats = 0;
  size_t slice_max = 0;
  for (const ChainOp& o : ops) {
    p.nb_max = o.nb > p.nb_max ? o.nb : p.nb_max;
    const int tq = o.epi ? 2 : 1;
    const size_t tiles = (size_t)tq * ceil_div(o.n_tiles / tq, grid);
    slice_max = std::max(slice_max, tiles * o.nb * kUnitBytes);
    if (o.epi) p.tv_floats = std::max(p.tv_floats, (int)(tiles * 64));
  }
  p.ng = batch <= 2 ? 1 : 2;
  p.nrx = batch <= 2 ? batch : 4;
  const size_t cap = 227 * 1024;
  const ChainSmem m0 = chain_smem(p.ng, p.nb_max, p.nrx, 0, p.tv_floats, (int)ops.size());
  size_t ring = m0.total < cap ? (cap - m0.total) / kUnitBytes * kUnitBytes : 0;
  if (ring_cap && ring > ring_cap) ring = ring_cap / kUnitBytes * kUnitBytes;
  if (ring < slice_max) {
    set_error("tr_linear_chain: a CTA's weight slice (%zu B) does not fit the %zu B ring next to %d staged blocks "
              "x batch %d", slice_max, ring, p.nb_max, batch);
    return -1;
  }
  p.ring_bytes = ring;
  p.smem = m0.total + ring;
  return 0;
}

// workspace: [counters 4 KiB | ChainOp table | ChainW table | trace (dev probe)]
static size_t chain_trace_off(int n_ops) {
  return ((size_t)kChainCounterBytes + (sizeof(ChainOp) + sizeof(ChainW)) * (size_t)n_ops + 255) / 256 * 256;
}
size_t chain_workspace_bytes(int n_ops) { return chain_trace_off(n_ops) + (size_t)n_ops * sm_count() * 16 * 8; }

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
  if (chain_plan(ops, batch, grid, p, (size_t)((flags >> 8) & 0xFF) * 4096)) return -1;   // (dev knob: ring cap)
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
  a.probe = (flags >> 24) & 0xF;
  a.ring_bytes = p.ring_bytes;
  a.piece = ((flags >> 16) & 0xFF) ? ((flags >> 16) & 0xFF) * 1024 : kChainPiece;   // (dev knob: KiB)
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
  cfg.blockDim = dim3((kChainWarps + 1) * 32, 1, 1);
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
  if (e != cudaSuccess) {
    int occ = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, (kChainWarps + 1) * 32, p.smem);
    cudaFuncAttributes fa = {};
    cudaFuncGetAttributes(&fa, kern);
    set_error("tr_linear_chain: launch failed: %s (grid %d, smem %zu, occupancy %d, regs %d, max dyn smem %d)",
              cudaGetErrorString(e), grid, p.smem, occ, fa.numRegs, fa.maxDynamicSharedSizeBytes);
    return -1;
  }
  return 0;
}

}  // namespace tr
