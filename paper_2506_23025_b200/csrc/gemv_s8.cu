// K3-S8: decode GEMV for batch 1-4 on the int8 tensor-core MMA, TQ2 weights.
//
// Semantics are K3's (reference linear.py:137-166, _kernels.pyx:136-168, paper App. F):
//   y[n, r] = sum_b s[r, b] * (sum_{k in block b} trit[r, k] * x[n, k]),
// inner block sums exact, scaled and accumulated in fp32, the output rounded once.
//
// Why int8: at batch 1-2 the fp16 mma.sync GEMV is issue-bound, not
// HBM-bound -- one LOP3 per half2 of weights plus 16 HMMA.16816 per 16x256 unit (measured:
// the kernel runs as fast with the weight stream switched off).  Here
//  * each activation block (256 columns, one batch row) is put on an integer grid:
//    x~ = rint(x * 2^(23-e)), 2^e <= max|x| < 2^(e+1), |x~| < 2^24 (fp16/bf16 values down to
//    2^-24 of the block maximum are exact, smaller ones carry an error below 2^-24 max|x|);
//  * column k's value is pre-multiplied by 4^(3-j), j = (k >> 2) & 3 its field class in the
//    T16 word, and split into 4 signed bytes (slices);
//  * a weight field is extracted by ONE LOP3 per FOUR weights: the byte (w >> 0) & (3 << 2j)
//    is the u8 4^j * d (d = trit + 1), so A = 4^j d and B = 4^(3-j) x~ multiply to 64 d x~ for
//    every class -- one int32 accumulator, exact;
//  * the 4 slices (x 2 batch rows) are the N = 8 columns of mma.sync.m16n8k32.u8.s8.s32, which
//    has the HMMA.16816's issue cost at twice the K: 8 IMMA + 32 LOP3 per unit instead of
//    16 HMMA + 64 LOP3 + 20 FFMA (batch 3-4: a second MMA group on the same A fragments);
//  * the trit offset is folded into the accumulator: the first MMA of a block starts from
//    -Cs, Cs[slice] = sum_k 4^j(k) b_slice(k), so D = sum_k 4^j (d - 1) b(k) exactly;
//  * per block: two slices combine in int32, one I2F + FFMA per row applies the block scale
//    and the block grid 2^(e-29); the two slice pairs meet by one shuffle when a tile closes.
// Weight streaming, tile ownership and the deterministic boundary-tile reduction are K3's.
#include "attn_core.cuh"
#include "s8_core.cuh"

namespace tr {

struct S8Args {
  const uint8_t* w;
  const void* x;
  void* y;
  int64_t ldx, ldy;
  int rows, cols, nb, n_tiles;
  int x_vec;
  int batch;   // 1 or 2
  int ns;      // ring slots per warp (power of two)
  int epi;       // 1: SwiGLU epilogue -- W rows are 16-row tiles alternating gate / up; the CTA
                 //    keeps its tile results in shared memory and stores silu(gate) * up (rows / 2)
  int cosched;   // co-scheduled with neighbouring GEMVs: half-SM CTAs (TR_LINEAR_COSCHEDULE)
  // development probes (tr_linear knob bits 12-15; 0 in production): 1 = 16 warps, 2 = per-CTA /
  // per-warp %globaltimer stamps into y (no output), 4 / 8 / 12 = ring issue order variants
  int dbg;
  int pre;     // fused producer of x (K3's GemvArgs::pre): 1 add+RMSNorm, 2 SwiGLU
  const void* pre_delta;
  const void* pre_gamma;
  void* pre_out;
  float eps;
  int out_f32;   // TR_LINEAR_OUT_F32: y is float32
  int fmt;       // kFmtTq2 (K3-S8) or kFmtTq1 (K4)
  // ATT = 1 (tr_qkv_attn_decode): y is one token's qkv [3, H, 128]; CTA b serves head b / (3 m): its
  // q, k or v section ((b % 3m) / m), 8 / m tiles of it; the head's last CTA to finish runs its attention
  const int64_t* att_pos;
  const void* att_cos;
  const void* att_sin;
  void* att_kc;
  void* att_vc;
  void* att_out;
  int att_heads, att_seq;
  float att_scale;
  unsigned* att_cnt;   // per-head arrival counters (zero between launches)
  int att_m;           // CTAs per q / k / v section of a head (1, 2, 4 or 8)
};

template <typename T, int NW, int PRE, int NG, int FMT = kFmtTq2, int ATT = 0>
__global__ void __launch_bounds__(NW * 32, NW == 8 ? 2 : 1) k_gemv_s8(const S8Args a) {
  static_assert(FMT == kFmtTq2 || PRE == 0, "fused producers are TQ2-only");
  using Cfg = S8Cfg<NW, NG, FMT>;
  constexpr int kSlotBytes = Cfg::kSlotBytes;
  constexpr int UB = S8Fmt<FMT>::kUnit;       // bytes per 16 x 256 unit
  constexpr int IB = S8Fmt<FMT>::kItem;       // staged bytes per (block, batch row)
  extern __shared__ __align__(128) uint8_t smem[];
  // batch rows nbr; staged layout rows nrx (1, 2, or 4 for NG = 2: batch 3-4), log2 lr
  const int NS = a.ns, nbr = a.batch, nb = a.nb;
  const int nrx = NG == 2 ? 4 : nbr, lr = NG == 2 ? 2 : nbr - 1;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                 // NW * NS <= 64
  int* slot_tile = reinterpret_cast<int*>(smem + 512);                 // 2 * NW
  float* red = reinterpret_cast<float*>(smem + Cfg::kRedOff);
  int32_t* ncs = reinterpret_cast<int32_t*>(smem + Cfg::kCsOff);
  float* fsc = reinterpret_cast<float*>(smem + Cfg::f_off(nb, nrx));
  uint8_t* xs = smem + Cfg::xs_off(nb, nrx);
  uint8_t* ring = smem + Cfg::ring_off(nb, nrx);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  uint64_t* mybar = bars + warp * NS;
  uint8_t* myring = ring + warp * NS * kSlotBytes;
  uint64_t* trace = (a.dbg & 2) ? reinterpret_cast<uint64_t*>(a.y) : nullptr;
  // (dev probe dbg&2) CTA stamps [blockIdx][0..7] = %globaltimer (ns); warp stamps
  // [148*8 + (blockIdx*NW + warp)*4 + k-8] = SM clock cycles since the warp left griddepcontrol.wait
  // (k = 8 staged, 9 main loop done, 10 stored, 11 first activation loads landed)
  long long wait_clk = 0;
  auto stamp = [&](int k) {
    if (trace && lane == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (k < 8) {
        if (warp == 0) trace[blockIdx.x * 8 + k] = t;
      } else {
        trace[148 * 8 + (blockIdx.x * NW + warp) * 4 + (k - 8)] = (uint64_t)(clock64() - wait_clk);
      }
    }
  };
  stamp(0);

  // the CTA owns whole tiles [t0, t1); warp w a contiguous slice of their units
  // (32-bit unsigned arithmetic: tiles x grid < 2^32 -- a 64-bit division here sat in front of
  // the first weight copies)
  // (SwiGLU epilogue: whole gate / up tile pairs per CTA)
  const unsigned tq = a.epi ? 2u : 1u, tn = (unsigned)a.n_tiles / tq;
  unsigned t0 = tq * (blockIdx.x * tn / gridDim.x);
  unsigned t1 = tq * ((blockIdx.x + 1) * tn / gridDim.x);
  if (ATT && !(a.dbg & 64)) {   // head-major: the 3 m CTAs of a head are neighbours in the grid (dbg 64: probe)
    const unsigned m = (unsigned)a.att_m, hh = blockIdx.x / (3u * m), r = blockIdx.x % (3u * m);
    t0 = (r / m) * 8u * (unsigned)a.att_heads + hh * 8u + (r % m) * (8u / m);
    t1 = t0 + 8u / m;
  }
  const int LL = (int)(t1 - t0) * nb;
  const int wu0 = (int)t0 * nb + (int)((unsigned)(warp * LL) / NW);
  const int wu1 = (int)t0 * nb + (int)((unsigned)((warp + 1) * LL) / NW);

  // ---- weight stream (lane 0): bulk copies of kS8SU units into the warp's ring
  int pu = wu0;
  uint64_t pol = 0;
  auto issue = [&](int slot) {
    if (pu >= wu1) return;
    const int n = min(kS8SU, wu1 - pu);
    mbar_expect_tx(&mybar[slot], n * UB);
    bulk_g2s(myring + slot * kSlotBytes, a.w + (int64_t)pu * UB, n * UB, &mybar[slot], pol);
    pu += n;
  };
  if (lane == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < NS; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
    slot_tile[2 * warp] = -1;
    slot_tile[2 * warp + 1] = -1;
  }
  // weights do not depend on the previous kernel: prefetch before griddepcontrol.wait
  // (dev knobs dbg&12: 4 = whole ring before the wait, 8 = one slot before and the rest after the
  // first activation loads, 12 = one slot before and the rest after staging)
  // Long per-warp ranges: only the first slot goes out before the wait -- the rest follows the
  // activation loads, which would otherwise queue behind a deep ring fill (measured: -4..-10% on
  // 9216x3072, 18432x3072, 11008x4096, 4096x11008; short ranges keep the whole ring in flight)
  const bool ring_after_staging = (a.dbg & 12) == 12;   // dev probe: one slot before, the rest after staging
  // (dbg&12 == 4: the whole ring before the wait, whatever the range)
  const int pre_slots = ((a.dbg & 12) == 4) ? NS : ((a.dbg & 8) || LL >= S8_PRE1_UNITS * NW) ? 1 : NS;
  if (lane == 0)
    for (int s = 0; s < pre_slots; ++s) issue(s);
  __syncwarp();
  if constexpr (FMT == kFmtTq1) {   // K4's B' slot table in the (still unused) reduction buffer
    s8q1_slot_table(reinterpret_cast<int*>(red));
    __syncthreads();
  }
  if constexpr (ATT) {   // the head's cached keys / values (written a decode step ago) -> L2 under the GEMV
    if (blockIdx.x % (3 * a.att_m) == 0 && threadIdx.x == 32 && !(a.dbg & 16)) {
      int ps = (int)*reinterpret_cast<const volatile int64_t*>(a.att_pos);   // speculative (see k_attn_decode)
      ps = ps < 0 ? 0 : (ps > a.att_seq ? a.att_seq : ps);
      if (ps > 0) {
        const int64_t off = (int64_t)(blockIdx.x / (3 * a.att_m)) * a.att_seq * 128 * sizeof(T);
        const uint32_t bytes = (uint32_t)ps * 128u * sizeof(T);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"((const uint8_t*)a.att_kc + off), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"((const uint8_t*)a.att_vc + off), "r"(bytes)
                     : "memory");
      }
    }
  }
  // RMSNorm producer: gamma is a parameter like the weights (not written by the previous kernel,
  // tr_linear_pre's contract), so this warp's first two gamma blocks load before the wait --
  // per layer they are the one HBM miss among the producer's inputs
  uint4 pgv[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
  if constexpr (PRE == 1) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int item = warp + i * NW;
      if (item < nb * nrx)
        pgv[i] = s8_load8(reinterpret_cast<const T*>(a.pre_gamma), (int64_t)(item >> lr) * kBlock + lane * 8, a.cols,
                          a.x_vec);
    }
  }
  if constexpr (!ATT) griddep_launch_dependents();   // (ATT: after the main loop, below)
  griddep_wait();   // x belongs to the previous kernel until here
  if (trace) wait_clk = clock64();
  stamp(1);
  // the rest of the ring is issued right after this warp's first activation loads, so those
  // loads are not queued behind the weight stream
  bool rest_issued = pre_slots >= NS || ring_after_staging;
  auto issue_rest = [&]() {
    if (!rest_issued) {
      if (lane == 0)
        for (int s = pre_slots; s < NS; ++s) issue(s);
      rest_issued = true;
    }
  };

  // ---- stage the activations as int8 slices (fused producer first when asked)
  const T* xg = reinterpret_cast<const T*>(a.x);

  if (PRE == 1) {   // x = rmsnorm(x + delta) * gamma; CTA 0 stores x + delta (the residual)
    float* ss_buf = red;   // nb * nrx partial sums of squares
    const T* gam = reinterpret_cast<const T*>(a.pre_gamma);
    // x and delta of this warp's first two blocks are loaded together up front (one memory latency
    // instead of one per block and pass); gamma (loaded before the wait) stays in registers for pass 2
    uint4 pxv[2], pdv[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int item = warp + i * NW;
      pxv[i] = pdv[i] = make_uint4(0, 0, 0, 0);
      if (item < nb * nrx) {
        const int kb = item >> lr, br = item & (nrx - 1);
        const int64_t kx = (int64_t)kb * kBlock + lane * 8;
        if (br < nbr) {
          pxv[i] = s8_load8(xg + br * a.ldx, kx, a.cols, a.x_vec);
          if (a.pre_delta) pdv[i] = s8_load8(reinterpret_cast<const T*>(a.pre_delta) + br * a.ldx, kx, a.cols, a.x_vec);
        }
      }
    }
    issue_rest();
    for (int item = warp, ii = 0; item < nb * nrx; item += NW, ++ii) {
      const int kb = item >> lr, br = item & (nrx - 1);
      const int64_t kx = (int64_t)kb * kBlock + lane * 8;
      float f[8];
      const bool live = br < nbr;   // (layout rows past the batch stage zeros)
      uint4 xv = ii == 0 ? pxv[0] : pxv[1], dv = ii == 0 ? pdv[0] : pdv[1];
      if (ii >= 2) {
        xv = live ? s8_load8(xg + br * a.ldx, kx, a.cols, a.x_vec) : make_uint4(0, 0, 0, 0);
        dv = make_uint4(0, 0, 0, 0);
        if (a.pre_delta && live)
          dv = s8_load8(reinterpret_cast<const T*>(a.pre_delta) + br * a.ldx, kx, a.cols, a.x_vec);
      }
      s8_f8<T>(xv, f);
      if (trace && ii == 0) {   // (dev probe: first loads landed)
        asm volatile("" ::"f"(f[0]));
        stamp(11);
      }
      if (a.pre_delta) {
        float d[8];
        s8_f8<T>(dv, d);
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = s8_rnd<T>(f[e] + d[e]);
      }
      const uint4 hv = s8_pack8<T>(f);
      *reinterpret_cast<uint4*>(xs + (size_t)item * kS8ItemBytes + lane * 16) = hv;   // parked in its own item
      if (blockIdx.x == 0 && a.pre_out && kx < a.cols && live) {
        T* o = reinterpret_cast<T*>(a.pre_out) + br * a.ldx + kx;
        if (kx + 8 <= a.cols && a.x_vec) {
          *reinterpret_cast<uint4*>(o) = hv;
        } else {
          const T* he = reinterpret_cast<const T*>(&hv);
          for (int e = 0; e < 8 && kx + e < a.cols; ++e) o[e] = he[e];
        }
      }
      float ss = 0.0f;
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += f[e] * f[e];
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) ss_buf[item] = ss;
    }
#ifdef S8_PRE_PROBE
    stamp(9);
#endif
    __syncthreads();
#ifdef S8_PRE_PROBE
    stamp(10);
#endif
    // inverse RMS of every staged row, once per warp before its items (the same fixed-order sum in
    // every warp and CTA; it was recomputed per item, a reduction chain in front of each staging)
    float ivr[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (r >= nrx) break;   // (warp-uniform)
      float ss = 0.0f;
      for (int q = lane; q < nb; q += 32) ss += ss_buf[q * nrx + r];
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      ivr[r] = rsqrtf(ss / a.cols + a.eps);
    }
    for (int item = warp, ii = 0; item < nb * nrx; item += NW, ++ii) {
      const int kb = item >> lr, br = item & (nrx - 1);
      const int64_t kx = (int64_t)kb * kBlock + lane * 8;
      float f[8], gm[8];
      s8_f8<T>(*reinterpret_cast<const uint4*>(xs + (size_t)item * kS8ItemBytes + lane * 16), f);
      s8_f8<T>(ii == 0 ? pgv[0] : ii == 1 ? pgv[1] : s8_load8(gam, kx, a.cols, a.x_vec), gm);
      const float iv = br == 0 ? ivr[0] : br == 1 ? ivr[1] : br == 2 ? ivr[2] : ivr[3];
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = s8_rnd<T>(s8_rnd<T>(f[e] * iv) * gm[e]);
      __syncwarp();   // every lane holds its h before the item's bytes are overwritten
      s8_stage_block(f, xs, ncs, fsc, nrx, kb, br);
    }
  } else {   // plain x, or silu(gate) * up of a gate|up product; loads for 4 items in flight
    const int n_items = nb * nrx;
    for (int i0 = warp; i0 < n_items; i0 += 4 * NW) {
      uint4 va[4], vb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int item = i0 + i * NW;
        if (item < n_items) {
          const int kb = item >> lr, br = item & (nrx - 1);
          const int64_t kx = (int64_t)kb * kBlock + lane * 8;
          const bool live = br < nbr;   // (layout rows past the batch stage zeros)
          va[i] = live ? s8_load8(xg + br * a.ldx, kx, a.cols, a.x_vec) : make_uint4(0, 0, 0, 0);
          if (PRE == 2) vb[i] = live ? s8_load8(xg + br * a.ldx + a.cols, kx, a.cols, a.x_vec) : make_uint4(0, 0, 0, 0);
        }
      }
      issue_rest();
#pragma unroll 1
      for (int i = 0; i < 4; i += 2) {   // two blocks per pass (their latency chains interleave)
        float f[2][8];
        int kbs[2], brs[2];
        int nv = 0;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int item = i0 + (i + t) * NW;
          const int it = item < n_items ? item : i0;
          kbs[t] = it >> lr;
          brs[t] = it & (nrx - 1);
          nv += item < n_items;
          s8_f8<T>(va[t], f[t]);
          if (trace && i0 == warp && i == 0 && t == 0) {   // (dev probe: first loads landed)
            asm volatile("" ::"f"(f[0][0]));
            stamp(11);
          }
          if (PRE == 2) {
            float up[8];
            s8_f8<T>(vb[t], up);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              f[t][e] = s8_rnd<T>(s8_rnd<T>(__fdividef(f[t][e], 1.0f + __expf(-f[t][e]))) * up[e]);   // (0 past cols)
          }
        }
        if constexpr (FMT == kFmtTq1) {
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (t < nv)
              s8q1_stage_block(f[t], xs + (size_t)(kbs[t] * nrx + brs[t]) * IB, ncs + (kbs[t] * nrx + brs[t]) * 4,
                               fsc + kbs[t] * nrx + brs[t], reinterpret_cast<const int*>(red));
        } else {
          if (nv > 0) s8_stage_blocks<2>(f, xs, ncs, fsc, nrx, kbs, brs, nv);
        }
        va[0] = va[2];
        va[1] = va[3];
        if (PRE == 2) {
          vb[0] = vb[2];
          vb[1] = vb[3];
        }
      }
    }
  }
  issue_rest();
  stamp(8);
  __syncthreads();
  if (ring_after_staging && lane == 0)
    for (int s = pre_slots; s < NS; ++s) issue(s);
  stamp(2);

  // ---- main loop: units [wu0, wu1), tile by tile
  // MMA group G2 covers batch rows 2 G2, 2 G2 + 1 (slice-columns 8 G2 .. 8 G2 + 7)
  T* y = reinterpret_cast<T*>(a.y);
  uint32_t xsB32[NG];
  const int32_t* ncsD[NG];
  const float* fscD[NG];
#pragma unroll
  for (int G2 = 0; G2 < NG; ++G2) {
    const int nBc = NG == 1 ? (g & (4 * nrx - 1)) : 8 * G2 + g;   // B column of this lane: slice-column
    const int bB = nBc >> 2, sB = nBc & 3;
    const int swB = ((c >> 1) << 1) | (sB & 1);
    // B fragment base in shared space: the group swizzle (q ^ swB) becomes an XOR on bits 4-5
    // (TQ1: the lane's 18 B' words of slice sB, lane column c)
    if constexpr (FMT == kFmtTq1)
      xsB32[G2] = smem_u32(xs + (size_t)bB * IB + (sB * 4 + c) * 80);
    else
      xsB32[G2] = smem_u32(xs + (size_t)bB * IB + sB * 256 + c * 64) ^ (uint32_t)(swB << 4);
    const int bD = NG == 1 ? min(c >> 1, nrx - 1) : 2 * G2 + (c >> 1);   // D: slices 2(c&1), +1 of this row
    ncsD[G2] = ncs + bD * 4 + 2 * (c & 1);
    fscD[G2] = fsc + bD;
  }
  const int kb_shift = 10 + lr;                // log2(nrx * kS8ItemBytes) (TQ2)
  const uint32_t kb_stride = (uint32_t)(nrx * IB);
  const float lane_w = (c & 1) ? 65536.0f : 1.0f;

  float* tv = reinterpret_cast<float*>(smem + Cfg::smem(nb, nrx, NS));   // (epi) [tile - t0][16 rows][4]
  auto store_tile = [&](int tile, const float (&v)[NG][2]) {
    if (trace) return;
    if (a.epi) {   // keep: the pair's other tile may come from another warp
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
        if (r0 < a.rows) store_y<T>(a.y, (int64_t)row * a.ldy + r0, v[G2][0], a.out_f32);
        if (r1 < a.rows) store_y<T>(a.y, (int64_t)row * a.ldy + r1, v[G2][1], a.out_f32);
      }
    }
  };
  const int first_tile = wu0 < wu1 ? wu0 / nb : -1;
  int cur = first_tile;
  float acc[NG][2];
#pragma unroll
  for (int G2 = 0; G2 < NG; ++G2) acc[G2][0] = acc[G2][1] = 0.0f;
  auto close_tile = [&](int tile) {   // combine the two slice pairs; store or park
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

  // The two units of a ring slot, interleaved: NG = 1: two accumulator chains of 8 IMMAs;
  // NG = 2: 32 IMMAs, two chains per unit (one per group).
  auto mma_pair = [&](const uint4 (&wl)[kS8SU], const uint4 (&wh)[kS8SU], const int (&kbq)[kS8SU],
                      int (&D)[kS8SU][NG][4]) {
    if constexpr (NG == 1) {
      uint4 xw[kS8SU][4];
      int2 cs[kS8SU];
#pragma unroll
      for (int q = 0; q < kS8SU; ++q) {
        const uint32_t xp = xsB32[0] + ((uint32_t)kbq[q] << kb_shift);
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) xw[q][i4] = ld_shared_v4u(xp ^ (i4 << 4));
        cs[q] = *reinterpret_cast<const int2*>(ncsD[0] + (kbq[q] << (lr + 2)));
      }
      int da[kS8SU][4], db[kS8SU][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int w = i >> 1, j0 = 2 * (i & 1);
        const uint32_t m0 = 0x03030303u << (2 * j0), m1 = 0x03030303u << (2 * j0 + 2);
#pragma unroll
        for (int q = 0; q < kS8SU; ++q) {
          const uint32_t lw = u4c(wl[q], w), hw = u4c(wh[q], w);
          const uint32_t A[4] = {lw & m0, hw & m0, lw & m1, hw & m1};
          const uint32_t b0 = u4c(xw[q][w], j0), b1 = u4c(xw[q][w], j0 + 1);
          if (i == 0)
            imma_c(da[q], A, b0, b1, cs[q].x, cs[q].y, cs[q].x, cs[q].y);
          else if (S8_TWO_CHAINS && i == 1)
            imma_c(db[q], A, b0, b1, 0, 0, 0, 0);
          else
            imma((S8_TWO_CHAINS && (i & 1)) ? db[q] : da[q], A, b0, b1);
        }
      }
#pragma unroll
      for (int q = 0; q < kS8SU; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) D[q][0][e] = S8_TWO_CHAINS ? da[q][e] + db[q][e] : da[q][e];
    } else {
#pragma unroll
      for (int q = 0; q < kS8SU; ++q) {
        uint4 xw[NG][4];
        int2 cs[NG];
#pragma unroll
        for (int G2 = 0; G2 < NG; ++G2) {
          const uint32_t xp = xsB32[G2] + ((uint32_t)kbq[q] << kb_shift);
#pragma unroll
          for (int i4 = 0; i4 < 4; ++i4) xw[G2][i4] = ld_shared_v4u(xp ^ (i4 << 4));
          cs[G2] = *reinterpret_cast<const int2*>(ncsD[G2] + (kbq[q] << (lr + 2)));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int w = i >> 1, j0 = 2 * (i & 1);
          const uint32_t m0 = 0x03030303u << (2 * j0), m1 = 0x03030303u << (2 * j0 + 2);
          const uint32_t lw = u4c(wl[q], w), hw = u4c(wh[q], w);
          const uint32_t A[4] = {lw & m0, hw & m0, lw & m1, hw & m1};
#pragma unroll
          for (int G2 = 0; G2 < NG; ++G2) {
            const uint32_t b0 = u4c(xw[G2][w], j0), b1 = u4c(xw[G2][w], j0 + 1);
            if (i == 0)
              imma_c(D[q][G2], A, b0, b1, cs[G2].x, cs[G2].y, cs[G2].x, cs[G2].y);
            else
              imma(D[q][G2], A, b0, b1);
          }
        }
      }
    }
  };
  auto epilogue = [&](const int (&d)[NG][4], uint32_t sv, int kbq) {   // block scale x grid, into the row sums
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
  const int nslog = NS == 1 ? 0 : NS == 2 ? 1 : 2;
  int k = 0;
#pragma unroll 1
  for (int u = wu0; u < wu1; ++k) {
    const int s = k & (NS - 1);
    const int n = min(kS8SU, wu1 - u);
    if (k > 0) {   // refill the slot read in the previous iteration (its loads have completed)
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async_smem();
        issue((k - 1) & (NS - 1));
      }
    }
    mbar_wait(&mybar[s], (k >> nslog) & 1);
    const uint8_t* slot = myring + s * kSlotBytes;
    if constexpr (FMT == kFmtTq1) {   // K4: units decoded by IMAD (F_k of both codes of a pair-group)
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
          const uint8_t* up = slot + q * UB;
          uint32_t xq[NG];
          int2 cs[NG];
#pragma unroll
          for (int G2 = 0; G2 < NG; ++G2) {
            xq[G2] = xsB32[G2] + (uint32_t)kb * kb_stride;
            cs[G2] = *reinterpret_cast<const int2*>(ncsD[G2] + (kb << (lr + 2)));
          }
          int D[NG][4];
          q1_unit_mma<NG>(up, g, c, xq, cs, D);
          epilogue(D, *reinterpret_cast<const uint32_t*>(up + kQ1TileBlockBytes + g * 4), kb);
          ++kb;
        }
      }
      u += n;
      continue;
    }
    uint4 wl[kS8SU], wh[kS8SU];
    uint32_t sv[kS8SU];
#pragma unroll
    for (int q = 0; q < kS8SU; ++q) {
      if (q < n) {
        wl[q] = lds128(slot + q * kUnitBytes + t16_word(0, c, g) * 16);
        wh[q] = lds128(slot + q * kUnitBytes + t16_word(1, c, g) * 16);
        sv[q] = *reinterpret_cast<const uint32_t*>(slot + q * kUnitBytes + kTileBlockBytes + g * 4);
      }
    }
    if (n == kS8SU && kb + kS8SU <= nb) {   // common case: a full slot inside one tile
      int kbq[kS8SU];
#pragma unroll
      for (int q = 0; q < kS8SU; ++q) kbq[q] = kb + q;
      int D[kS8SU][NG][4];
      mma_pair(wl, wh, kbq, D);
#pragma unroll
      for (int q = 0; q < kS8SU; ++q) epilogue(D[q], sv[q], kbq[q]);
      kb += kS8SU;
      u += n;
      continue;
    }
    // blocks of the slot's units (a partial last slot recomputes unit 0 and drops it)
    int kbq[kS8SU];
    bool wrap[kS8SU];
#pragma unroll
    for (int q = 0; q < kS8SU; ++q) {
      wrap[q] = q < n && kb == nb;
      if (wrap[q]) kb = 0;
      kbq[q] = q < n ? kb : kbq[0];
      if (q < n) ++kb;
      if (q >= n) {
        wl[q] = wl[0];
        wh[q] = wh[0];
      }
    }
    int D[kS8SU][NG][4];
    mma_pair(wl, wh, kbq, D);
#pragma unroll
    for (int q = 0; q < kS8SU; ++q) {
      if (q < n) {
        if (wrap[q]) {   // next tile
          close_tile(cur);
#pragma unroll
          for (int G2 = 0; G2 < NG; ++G2) acc[G2][0] = acc[G2][1] = 0.0f;
          ++cur;
        }
        epilogue(D[q], sv[q], kbq[q]);
      }
    }
    u += n;
  }
#ifndef S8_PRE_PROBE
  stamp(9);
#endif
  // the fused QKV + attention kernel lets the o projection launch only once its GEMV part is done:
  // its 16-warp CTAs and the attention tail otherwise share the SMs with waiting o-projection CTAs
  if constexpr (ATT) griddep_launch_dependents();
  if (cur >= 0) close_tile(cur);

  // ---- boundary tiles: combine the parked fragments in fixed (warp, slot) order and store
  __syncthreads();
  const int my_tag = lane < 2 * NW ? slot_tile[lane] : -1;
  for (int i = warp; i < 2 * NW; i += NW) {
    const int tile = __shfl_sync(0xffffffffu, my_tag, i);
    if (tile < 0) continue;
    const unsigned match = __ballot_sync(0xffffffffu, my_tag == tile);
    if (match & ((1u << i) - 1u)) continue;   // a lower slot holds this tile: it reduces
    float v[NG][2];
#pragma unroll
    for (int G2 = 0; G2 < NG; ++G2) v[G2][0] = v[G2][1] = 0.0f;
    for (unsigned mq = match; mq; mq &= mq - 1) {   // ascending slot order: deterministic
      const int q = __ffs(mq) - 1;
#pragma unroll
      for (int G2 = 0; G2 < NG; ++G2) {
        v[G2][0] += red[q * 64 * NG + G2 * 64 + lane];
        v[G2][1] += red[q * 64 * NG + G2 * 64 + 32 + lane];
      }
    }
    store_tile(tile, v);
  }
  if (a.epi) {   // silu(gate) * up with the roundings of the unfused gate|up store + tr_silu_mul
    __syncthreads();
    const int npairs = (int)(t1 - t0) / 2, rows_out = a.rows / 2;
    for (int idx = threadIdx.x; idx < npairs * 16 * nbr; idx += NW * 32) {
      const int p = idx / (16 * nbr), r = (idx / nbr) % 16, br = idx % nbr;
      const float gt = s8_rnd<T>(tv[(size_t)(2 * p) * 64 + r * 4 + br]);
      const float up = s8_rnd<T>(tv[(size_t)(2 * p + 1) * 64 + r * 4 + br]);
      const int orow = ((int)t0 / 2 + p) * 16 + r;
      if (orow < rows_out && !trace)
        y[br * a.ldy + orow] = Act<T>::from_float(s8_rnd<T>(__fdividef(gt, 1.0f + __expf(-gt))) * up);
    }
  }
#ifndef S8_PRE_PROBE
  stamp(10);
#endif
  if (warp == 0) stamp(3);
  if constexpr (ATT) {   // the last of the head's 3 m CTAs to store its rows runs the head's attention
    volatile int& last = slot_tile[0];   // (free by now; a static __shared__ would eat into the 227 KB opt-in)
    const unsigned hh = blockIdx.x / (3u * (unsigned)a.att_m);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned c;
      asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;\n" : "=r"(c) : "l"(a.att_cnt + hh) : "memory");
      last = c == 3u * (unsigned)a.att_m - 1u;
      if (last) a.att_cnt[hh] = 0;   // (all arrivals are in; the next launch reads it after griddepcontrol.wait)
    }
    __syncthreads();
    if (last && threadIdx.x < 128)
      attn::attn_head_128<T>(reinterpret_cast<const T*>(a.y), a.att_pos, reinterpret_cast<const T*>(a.att_cos),
                             reinterpret_cast<const T*>(a.att_sin), reinterpret_cast<T*>(a.att_kc),
                             reinterpret_cast<T*>(a.att_vc), reinterpret_cast<T*>(a.att_out), a.att_heads, a.att_seq,
                             (int)hh, a.att_scale, xs, threadIdx.x, 2);
  }
}

// ------------------------------------------------------------------------------------ host

#ifndef S8_NS16
#define S8_NS16 2   // weight-ring slots per warp at 16 warps (measured: decode 1114 -> 1128 tok/s; the
                    // BASELINE stack and the 70B layers within 0.5%)
#endif
template <int NW>
static int s8_ns(int n_tiles, int nb, int grid) {
  const int tiles_max = (int)ceil_div(n_tiles, grid);
  const int ops = (int)ceil_div(ceil_div((int64_t)tiles_max * nb, NW), kS8SU);
  const int cap = NW == 16 ? S8_NS16 : kS8NSMax;
  return ops >= cap ? cap : ops > 2 ? 4 : ops > 1 ? 2 : 1;
}

#ifndef S8_SMALL_UNITS
#define S8_SMALL_UNITS 48
#endif
constexpr int kS8SmallCtaUnits = S8_SMALL_UNITS;   // units per CTA at or below which 8 warps x 2 CTAs/SM are used

// 8 warps x 2 CTAs per SM (the next PDL-chained layer co-resides and prefetches) win for short
// per-CTA ranges, and up to 80 units while staging stays cheap (<= 16 blocks: <= 2 per warp);
// measured on the BASELINE and decoder shapes (scripts/dev/gpu53.sh)
static bool s8_small(int n_tiles, int nb, int grid) {
  const int64_t units = (int64_t)ceil_div(n_tiles, grid) * nb;
  return units <= kS8SmallCtaUnits || (units <= 80 && nb <= 16);
}

static int s8_layout_rows(int batch) { return batch <= 2 ? batch : 4; }   // staged rows (NG = 2 pads to 4)

template <int NW, int NG, int FMT = kFmtTq2>
static size_t s8_smem_plan(int batch, int nb, int n_tiles, int grid, int* ns_out, size_t cap = 227 * 1024) {
  int ns = s8_ns<NW>(n_tiles, nb, grid);
  const int nra = s8_layout_rows(batch);
  size_t sm = S8Cfg<NW, NG, FMT>::smem(nb, nra, ns);
  while (sm > cap && ns > 1) {   // wide activations: a shallower weight ring
    ns >>= 1;
    sm = S8Cfg<NW, NG, FMT>::smem(nb, nra, ns);
  }
  if (ns_out) *ns_out = ns;
  return sm;
}

template <int NG, int FMT>
static bool s8_fits_ng(int batch, int nb, int n_tiles, int grid) {
  int ns = 0;
  const size_t sm = s8_small(n_tiles, nb, grid) ? s8_smem_plan<8, NG, FMT>(batch, nb, n_tiles, grid, &ns)
                                                : s8_smem_plan<16, NG, FMT>(batch, nb, n_tiles, grid, &ns);
  return sm <= 227 * 1024 && (ns >= 2 || s8_ns<16>(n_tiles, nb, grid) < 2);
}

// true when the int8-slice GEMV (TQ2: K3-S8, TQ1: K4) takes this product (batch 1-4, activations
// fit with a weight ring of >= 2 slots)
bool gemv_s8_fits(int batch, int rows, int cols, int fmt) {
  if (batch < 1 || batch > 4) return false;
  const int nb = (int)ceil_div(cols, kBlock), n_tiles = (int)ceil_div(rows, 16);
  const int grid = sm_count() < n_tiles ? sm_count() : n_tiles;
  if (fmt == kFmtTq1)
    return batch <= 2 ? s8_fits_ng<1, kFmtTq1>(batch, nb, n_tiles, grid) : s8_fits_ng<2, kFmtTq1>(batch, nb, n_tiles, grid);
  return batch <= 2 ? s8_fits_ng<1, kFmtTq2>(batch, nb, n_tiles, grid) : s8_fits_ng<2, kFmtTq2>(batch, nb, n_tiles, grid);
}

static size_t s8_tv_bytes(const S8Args& a, int grid) {   // SwiGLU epilogue: tile results of one CTA
  return a.epi ? (size_t)2 * ceil_div(a.n_tiles / 2, grid) * 64 * sizeof(float) : 0;
}

template <typename T, int NW, int PRE, int NG, int FMT = kFmtTq2>
static int launch_s8_k(S8Args& a, int grid, int pdl, cudaStream_t st) {
  auto kern = k_gemv_s8<T, NW, PRE, NG, FMT>;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured_dev = dev;
  }
  const size_t smem =
      s8_smem_plan<NW, NG, FMT>(a.batch, a.nb, a.n_tiles, grid, &a.ns, 227 * 1024 - s8_tv_bytes(a, grid)) +
      s8_tv_bytes(a, grid);
  if (smem > 227 * 1024) {
    set_error("tr_linear(gemv-s8): %d blocks per row x batch %d need %zu B of shared memory", a.nb, a.batch, smem);
    return -1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(NW * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) {
    set_error("tr_linear(gemv-s8): launch failed: %s (grid %d, smem %zu)", cudaGetErrorString(e), grid, smem);
    return -1;
  }
  return 0;
}
template <typename T, int NW, int NG>
static int launch_s8_ng(S8Args& a, int grid, int pdl, cudaStream_t st) {   // one kernel per fused producer
  if (a.fmt == kFmtTq1) return launch_s8_k<T, NW, 0, NG, kFmtTq1>(a, grid, pdl, st);
  if (a.pre == 1) return launch_s8_k<T, NW, 1, NG>(a, grid, pdl, st);
  if (a.pre == 2) return launch_s8_k<T, NW, 2, NG>(a, grid, pdl, st);
  return launch_s8_k<T, NW, 0, NG>(a, grid, pdl, st);
}
template <typename T, int NW>
static int launch_s8(S8Args& a, int grid, int pdl, cudaStream_t st) {
  return a.batch <= 2 ? launch_s8_ng<T, NW, 1>(a, grid, pdl, st) : launch_s8_ng<T, NW, 2>(a, grid, pdl, st);
}

// Fused decode QKV projection + attention (tr_qkv_attn_decode): the add + RMSNorm producer and the
// int8-slice GEMV of K3-S8 with the tiles dealt head-major (3 m CTAs per head, each inside one of its
// q / k / v sections); each CTA counts itself in (atom.acq_rel) and the head's last CTA runs that
// head's attention, so no separate attention kernel -- and no kernel boundary -- follows the
// projection.  (Measured: the head-major deal beats the plain even split over all SMs, where every
// head waits on CTAs from three distant parts of the grid.)
template <typename T, int NW>
static int launch_qkv_attn(S8Args& a, int pdl, cudaStream_t st) {
  auto kern = k_gemv_s8<T, NW, 1, 1, kFmtTq2, 1>;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    TR_REQUIRE(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) == cudaSuccess,
               "tr_qkv_attn_decode: cannot opt in to 227 KB of shared memory");
    configured_dev = dev;
  }
  // m CTAs per q / k / v section of a head: the largest of 8, 4, 2, 1 with 3 m H CTAs in one wave
  // (H = 24: m = 2, 144 CTAs of 4 tiles; more heads than 49 run 3 H CTAs in several waves)
  int m = 8;
  while (m > 1 && 3 * m * a.att_heads > sm_count()) m >>= 1;
  a.att_m = m;
  const int grid = 3 * m * a.att_heads;
  const size_t smem = s8_smem_plan<NW, 1, kFmtTq2>(1, a.nb, a.n_tiles, grid, &a.ns);
  const size_t att_need = S8Cfg<NW, 1, kFmtTq2>::xs_off(a.nb, 1) + attn::kSmemBytes;
  const size_t smem_all = smem > att_need ? smem : att_need;
  TR_REQUIRE(smem_all <= 227 * 1024, "tr_qkv_attn_decode: %zu B of shared memory", smem_all);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(NW * 32, 1, 1);
  cfg.dynamicSmemBytes = smem_all;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  TR_REQUIRE(e == cudaSuccess, "tr_qkv_attn_decode: launch failed: %s (grid %d, smem %zu)", cudaGetErrorString(e),
             grid, smem_all);
  return 0;
}

int gemv_qkv_attn(int act, const void* w, const void* h, const void* delta, const void* gamma, void* h_out,
                  float eps, void* qkv, const int64_t* pos, const void* cos_t, const void* sin_t, void* k_cache,
                  void* v_cache, void* att_out, int heads, int head_dim, int max_seq, float scale, void* counters,
                  int pdl, int dbg, cudaStream_t st) {
  TR_REQUIRE(head_dim == 128, "tr_qkv_attn_decode: head_dim must be 128");
  TR_REQUIRE(heads >= 1 && max_seq >= 1 && max_seq <= 128, "tr_qkv_attn_decode: 1 <= max_seq <= 128");
  TR_REQUIRE(gamma != nullptr && h_out != nullptr, "tr_qkv_attn_decode: RMSNorm needs gamma and the residual output");
  const int d = heads * head_dim;
  S8Args a = {};
  a.fmt = kFmtTq2;
  a.w = (const uint8_t*)w;
  a.x = h;
  a.y = qkv;
  a.ldx = d;
  a.ldy = 3 * d;
  a.rows = 3 * d;
  a.cols = d;
  a.nb = (int)ceil_div(d, kBlock);
  a.n_tiles = (int)ceil_div(3 * d, 16);
  a.x_vec = (((uintptr_t)h | (uintptr_t)(delta ? delta : h) | (uintptr_t)gamma | (uintptr_t)h_out) % 16) == 0 ? 1 : 0;
  a.batch = 1;
  a.pre = 1;
  a.pre_delta = delta;
  a.pre_gamma = gamma;
  a.pre_out = h_out;
  a.eps = eps;
  a.att_pos = pos;
  a.att_cos = cos_t;
  a.att_sin = sin_t;
  a.att_kc = k_cache;
  a.att_vc = v_cache;
  a.att_out = att_out;
  a.att_heads = heads;
  a.att_seq = max_seq;
  a.att_scale = scale;
  a.dbg = dbg;
  a.att_cnt = (unsigned*)counters;
  TR_REQUIRE(counters != nullptr, "tr_qkv_attn_decode: needs the zeroed counter workspace");
  if (dbg & 256)   // dev probe: 8 warps
    return act == kActF16 ? launch_qkv_attn<__half, 8>(a, pdl, st) : launch_qkv_attn<__nv_bfloat16, 8>(a, pdl, st);
  return act == kActF16 ? launch_qkv_attn<__half, 16>(a, pdl, st) : launch_qkv_attn<__nv_bfloat16, 16>(a, pdl, st);
}

int gemv_s8(int act, const void* w, const void* x, void* y, int64_t ldx, int64_t ldy, int batch, int rows, int cols,
            int ctas, int pdl, cudaStream_t st, int pre, const void* pre_delta, const void* pre_gamma, void* pre_out,
            float eps, int cosched, int epi, int out_f32, int fmt) {
  if (!gemv_s8_fits(batch, rows, cols, fmt)) {
    set_error("tr_linear(gemv-s8): batch %d x %d columns does not fit the int8-slice GEMV", batch, cols);
    return -1;
  }
  if (fmt == kFmtTq1 && (pre || epi)) {
    set_error("tr_linear(gemv-q1): fused producers / epilogues run on TQ2 weights only");
    return -1;
  }
  S8Args a = {};
  a.fmt = fmt;
  a.w = (const uint8_t*)w;
  a.x = x;
  a.y = y;
  a.ldx = ldx;
  a.ldy = ldy;
  a.rows = rows;
  a.cols = cols;
  a.nb = (int)ceil_div(cols, kBlock);
  a.n_tiles = (int)ceil_div(rows, 16);
  a.x_vec = ((ldx % 8) == 0 && ((uintptr_t)x % 16) == 0) ? 1 : 0;
  a.batch = batch;
  a.pre = pre;
  a.pre_delta = pre_delta;
  a.pre_gamma = pre_gamma;
  a.pre_out = pre_out;
  a.eps = eps;
  a.dbg = (ctas >> 12) & 0xF;
  ctas &= 0xFFF;
  a.epi = epi;
  a.out_f32 = out_f32;
  if (epi && (rows % 32) != 0) {
    set_error("tr_linear(swiglu epilogue): rows (%d) must be whole 16-row gate/up tile pairs", rows);
    return -1;
  }
  int grid = ctas > 0 ? ctas : sm_count();
  const int units_of_work = epi ? a.n_tiles / 2 : a.n_tiles;   // (tile pairs for the SwiGLU epilogue)
  if (grid > units_of_work) grid = units_of_work;
  const bool bf = act != kActF16;
  a.cosched = cosched == 1;   // 8-warp CTAs (two per SM when their shared memory allows); 2: 16 warps
  // batch >= 2 stages two or four activation rows per block, and sixteen warps halve each warp's
  // share of that serial staging: they win whatever the co-scheduling (BASELINE stack, us per
  // layer: b=2 8.05 -> 6.71, b=3 10.09 -> 9.17, b=4 13.02 -> 11.79; b=1 stays with 8 warps,
  // 6.08 vs 6.12; scripts/dev/nw_probe.py)
  if (batch == 1 && cosched != 2 && (a.cosched || (s8_small(a.n_tiles, a.nb, grid) && !(a.dbg & 1))))   // (dev knob dbg&1: 16 warps)
    return bf ? launch_s8<__nv_bfloat16, 8>(a, grid, pdl, st) : launch_s8<__half, 8>(a, grid, pdl, st);
  return bf ? launch_s8<__nv_bfloat16, 16>(a, grid, pdl, st) : launch_s8<__half, 16>(a, grid, pdl, st);
}

}  // namespace tr
