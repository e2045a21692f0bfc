// Decoder-layer glue around the ternary linears (BASELINE configs[2]):
// one kernel each for residual-add + RMSNorm, rotary embedding + KV-cache append,
// single-token attention over the cache, and SwiGLU.  These are not part of the reference
// package (it has no model code); they exist so a decode step is ~8 launches per layer
// instead of ~50 PyTorch ops, and are used identically by the ternary model and its fp16
// cuBLAS twin (decoder.py).  All are HBM/latency-trivial: a few KB per launch.
#include "common.cuh"

namespace tr {

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float s = 0.0f;
  for (int i = 0; i < nw; ++i) s += red[i];   // fixed order: deterministic
  return s;
}

// h[r] += delta[r] (if delta); y[r] = h[r] * rsqrt(mean(h[r]^2) + eps) * w   (one CTA per row)
// Latency-bound (a 3072-wide row is 6 KB): every thread issues its 16-byte loads of h,
// delta and w up front, then one block reduction.
template <typename T>
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = to_f(e[i]);
}
template <typename T>
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  T* e = reinterpret_cast<T*>(&v);
#pragma unroll
  for (int i = 0; i < 8; ++i) e[i] = Act<T>::from_float(f[i]);
  return v;
}

template <typename T, int V>   // V: 8-element vectors per thread
__global__ void k_add_rmsnorm(T* __restrict__ h, const T* __restrict__ delta, const T* __restrict__ w,
                              T* __restrict__ y, int d, float eps) {
  griddep_wait();   // PDL: inputs come from the previous kernel
  griddep_launch_dependents();
  __shared__ float red[32];
  uint4* hr = reinterpret_cast<uint4*>(h + (int64_t)blockIdx.x * d);
  const uint4* dr = delta ? reinterpret_cast<const uint4*>(delta + (int64_t)blockIdx.x * d) : nullptr;
  uint4* yr = reinterpret_cast<uint4*>(y + (int64_t)blockIdx.x * d);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  const int nv = d / 8;
  uint4 hv[V], dv[V], wv[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < nv) {
      hv[j] = hr[i];
      wv[j] = wr[i];
      if (dr) dv[j] = dr[i];
    }
  }
  float ss = 0.0f;
  float hf[V][8];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < nv) {
      unpack8<T>(hv[j], hf[j]);
      if (dr) {
        float df[8];
        unpack8<T>(dv[j], df);
#pragma unroll
        for (int e = 0; e < 8; ++e) hf[j][e] += df[e];
        hv[j] = pack8<T>(hf[j]);
        hr[i] = hv[j];
        unpack8<T>(hv[j], hf[j]);   // the stored (rounded) residual is what the next layer sees
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += hf[j][e] * hf[j][e];
    }
  }
  const float inv = rsqrtf(block_sum(ss, red) / d + eps);
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < nv) {
      float wf[8], o[8];
      unpack8<T>(wv[j], wf);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = to_f(Act<T>::from_float(hf[j][e] * inv)) * wf[e];
      yr[i] = pack8<T>(o);
    }
  }
}

// qkv [T, 3, H, D] -> q [T, H, D] (rotated); rotated k and v written to the caches
// [H, S, D] at position pos[t].  Interleaved pairs (2i, 2i+1), angle cos/sin [S, D/2].
template <typename T>
__global__ void k_rope_kv(const T* __restrict__ qkv, const int64_t* __restrict__ pos, const T* __restrict__ cs,
                          const T* __restrict__ sn, T* __restrict__ q, T* __restrict__ kc, T* __restrict__ vc,
                          int H, int D, int S) {
  griddep_wait();   // PDL: inputs come from the previous kernel
  griddep_launch_dependents();
  const int t = blockIdx.y, hh = blockIdx.x;
  const int64_t p = pos[t];
  if (p < 0 || p >= S) return;   // past the cache (callers bound pos on the host too): write nothing
  const T* base = qkv + (int64_t)t * 3 * H * D;
  for (int i = threadIdx.x; i < D / 2; i += blockDim.x) {
    const float c = to_f(cs[p * (D / 2) + i]), s = to_f(sn[p * (D / 2) + i]);
    const float q1 = to_f(base[hh * D + 2 * i]), q2 = to_f(base[hh * D + 2 * i + 1]);
    const float k1 = to_f(base[(H + hh) * D + 2 * i]), k2 = to_f(base[(H + hh) * D + 2 * i + 1]);
    T* qo = q + ((int64_t)t * H + hh) * D;
    qo[2 * i] = Act<T>::from_float(q1 * c - q2 * s);
    qo[2 * i + 1] = Act<T>::from_float(q1 * s + q2 * c);
    T* ko = kc + ((int64_t)hh * S + p) * D;
    ko[2 * i] = Act<T>::from_float(k1 * c - k2 * s);
    ko[2 * i + 1] = Act<T>::from_float(k1 * s + k2 * c);
    T* vo = vc + ((int64_t)hh * S + p) * D;
    vo[2 * i] = base[(2 * H + hh) * D + 2 * i];
    vo[2 * i + 1] = base[(2 * H + hh) * D + 2 * i + 1];
  }
}

// One decode token, fused: rotary q/k of head hh from qkv [3, H, D], k/v appended to the
// caches [H, S, D] at pos, then out[hh] = softmax(q k^T * scale over keys 0..pos) v.
// One CTA (128 threads) per head.  Right after griddepcontrol.wait every load is issued at
// once -- this token's q/k/v, thread t's cached key t (16-byte loads into registers) and all
// cached values (cp.async into shared memory) -- so the kernel pays one memory latency, not
// three.  Thread t scores key t; the value sum is split over the 4 warps (lanes cover D) and
// combined in fixed order.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <typename T, int D>
__global__ void __launch_bounds__(128) k_attn_decode(const T* __restrict__ qkv, const int64_t* __restrict__ pos,
                                                     const T* __restrict__ cs, const T* __restrict__ sn,
                                                     T* __restrict__ kc, T* __restrict__ vc, T* __restrict__ out,
                                                     int H, int S, float scale) {
  static_assert(D == 128, "one key per thread, 4 dims per lane");
  {   // batched decode (tr_attn_decode_batch): sequence blockIdx.y -- its qkv row, position, caches, output
    const int64_t bq = blockIdx.y;
    qkv += bq * 3 * H * D;
    pos += bq;
    kc += bq * H * S * D;
    vc += bq * H * S * D;
    out += bq * H * D;
  }
  __shared__ __align__(16) T vs[128][D];   // values of keys 0..pos
  __shared__ __align__(16) T kp[D];        // this token's rotated key
  __shared__ float qs[D];
  __shared__ float sc[128];
  __shared__ float part[4][D];
  __shared__ float red[32];
  const int hh = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const T* kb = kc + (int64_t)hh * S * D;
  const T* vb = vc + (int64_t)hh * S * D;
  // cached values [lo, hi) -> shared memory (asynchronous), cached key tid -> registers.  Each
  // thread owns fixed chunks (c = tid mod 128), so a thread can top up its own range.
  uint4 kv[D / 8];
  auto load_cache = [&](int lo, int hi) {
    for (int c = lo * (D / 8) + tid; c < hi * (D / 8); c += 128)
      cp_async16(&vs[c / (D / 8)][(c % (D / 8)) * 8], vb + (int64_t)c * 8);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    if (tid >= lo && tid < hi) {
      const uint4* kr = reinterpret_cast<const uint4*>(kb + (int64_t)tid * D);
#pragma unroll
      for (int j = 0; j < D / 8; ++j) kv[j] = kr[j];
    }
  };
  // The cache rows before this token were written a whole decode step ago, so they load before
  // griddepcontrol.wait, under the QKV GEMV's tail.  pos itself may still be in flight (layer 0:
  // the previous step's greedy kernel can overlap through the PDL chain), so it is read again
  // after the wait and the missing rows are topped up; pos never decreases while a chain is in
  // flight (reset() is stream-ordered), so the speculative range is a prefix of the real one.
  int p_spec = (int)*reinterpret_cast<const volatile int64_t*>(pos);
  p_spec = p_spec < 0 ? 0 : (p_spec > S - 1 ? S - 1 : p_spec);
  load_cache(0, p_spec);
  // the rotary angles of the speculative position are parameters too: load them under the wait
  T cs_spec = Act<T>::from_float(0.0f), sn_spec = cs_spec;
  if (tid < D / 2) {
    cs_spec = cs[(int64_t)p_spec * (D / 2) + tid];
    sn_spec = sn[(int64_t)p_spec * (D / 2) + tid];
  }
  griddep_wait();
  griddep_launch_dependents();
  // this token's q / k / v and pos in one round trip (the q / k / v loads do not wait for pos)
  T qa = cs_spec, qb = cs_spec, ka = cs_spec, kb2 = cs_spec, v1 = cs_spec, v2 = cs_spec;
  if (tid < D / 2) {
    qa = qkv[hh * D + 2 * tid];
    qb = qkv[hh * D + 2 * tid + 1];
    ka = qkv[(H + hh) * D + 2 * tid];
    kb2 = qkv[(H + hh) * D + 2 * tid + 1];
    v1 = qkv[(2 * H + hh) * D + 2 * tid];
    v2 = qkv[(2 * H + hh) * D + 2 * tid + 1];
  }
  const int64_t p64 = pos[0];
  if (p64 < 0 || p64 >= S) {   // past the cache: no cache or shared-memory row p exists; output zeros
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    out[(int64_t)hh * D + tid] = Act<T>::from_float(0.0f);
    return;
  }
  const int p = (int)p64, n = p + 1;
  if (p > p_spec) load_cache(p_spec, p);
  // rotary embedding of this token's q and k; k and v into the caches (and shared memory)
  if (tid < D / 2) {
    const float c = to_f(p == p_spec ? cs_spec : cs[(int64_t)p * (D / 2) + tid]);
    const float s = to_f(p == p_spec ? sn_spec : sn[(int64_t)p * (D / 2) + tid]);
    const float q1 = to_f(qa), q2 = to_f(qb);
    const float k1 = to_f(ka), k2 = to_f(kb2);
    qs[2 * tid] = to_f(Act<T>::from_float(q1 * c - q2 * s));
    qs[2 * tid + 1] = to_f(Act<T>::from_float(q1 * s + q2 * c));
    const T r1 = Act<T>::from_float(k1 * c - k2 * s), r2 = Act<T>::from_float(k1 * s + k2 * c);
    kp[2 * tid] = r1;
    kp[2 * tid + 1] = r2;
    vs[p][2 * tid] = v1;
    vs[p][2 * tid + 1] = v2;
    T* ko = kc + ((int64_t)hh * S + p) * D;
    ko[2 * tid] = r1;
    ko[2 * tid + 1] = r2;
    T* vo = vc + ((int64_t)hh * S + p) * D;
    vo[2 * tid] = v1;
    vo[2 * tid + 1] = v2;
  }
  __syncthreads();
  // scores: thread tid <-> key tid (this token's key from shared memory)
  float v = -INFINITY;
  if (tid <= p) {
    if (tid == p) {
#pragma unroll
      for (int j = 0; j < D / 8; ++j) kv[j] = reinterpret_cast<const uint4*>(kp)[j];
    }
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      float kf[8];
      unpack8<T>(kv[j], kf);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc += qs[8 * j + e] * kf[e];
    }
    v = acc * scale;
  }
  float m = v;
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  const float e = tid < n ? __expf(v - m) : 0.0f;
  sc[tid] = e;
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");   // (block_sum syncs: values visible after it)
  const float z = block_sum(e, red);
  // value sum: warp w takes keys w, w+4, ...; lane covers dims 4 lane .. 4 lane + 3
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int s0 = warp; s0 < n; s0 += 4) {
    const uint2 vv = *reinterpret_cast<const uint2*>(&vs[s0][4 * lane]);
    const T* ve = reinterpret_cast<const T*>(&vv);
    const float w = sc[s0];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += w * to_f(ve[q]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) part[warp][4 * lane + q] = acc[q];
  __syncthreads();
  const float r = ((part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid])) / z;
  out[(int64_t)hh * D + tid] = Act<T>::from_float(r);
}

// Long caches (max_seq > 128): split-KV decode attention.  CTA (head hh, chunk c) scores keys
// [128 c, 128 c + 128) ∩ [0, pos] (thread t <-> key 128 c + t) and leaves a partial softmax
// {max, sum, sum_k e_k v_k[0..D)} in the workspace; the CTA whose chunk holds pos also rotates
// this token's key and appends k/v to the caches.  k_attn_combine merges the partials of a head
// (rescaling each by exp(m_c - M)).  Same roundings as k_attn_decode for q, k and the output.
template <typename T, int D>
__global__ void __launch_bounds__(128) k_attn_split(const T* __restrict__ qkv, const int64_t* __restrict__ pos,
                                                    const T* __restrict__ cs, const T* __restrict__ sn,
                                                    T* __restrict__ kc, T* __restrict__ vc, float* __restrict__ ws,
                                                    int H, int S, float scale) {
  static_assert(D == 128, "one key per thread, 4 dims per lane");
  __shared__ __align__(16) T vs[128][D];
  __shared__ __align__(16) T kp[D];
  __shared__ float qs[D];
  __shared__ float sc[128];
  __shared__ float part[4][D];
  __shared__ float red[32];
  const int hh = blockIdx.x, ch = blockIdx.y, NC = gridDim.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* wp = ws + ((int64_t)hh * NC + ch) * (D + 2);
  griddep_wait();
  griddep_launch_dependents();
  const int64_t p64 = pos[0];
  const int c0 = ch * 128;
  if (p64 < 0 || p64 >= S || c0 > p64) {   // no keys of this chunk are live (or pos is past the cache)
    if (tid == 0) {
      wp[0] = -INFINITY;
      wp[1] = 0.0f;
    }
    wp[2 + tid] = 0.0f;
    return;
  }
  const int p = (int)p64;
  const int nk = (p - c0 + 1) < 128 ? (p - c0 + 1) : 128;   // live keys in this chunk
  const bool own = p - c0 < 128;                              // this chunk holds the token itself
  const T* kb = kc + ((int64_t)hh * S + c0) * D;
  const T* vb = vc + ((int64_t)hh * S + c0) * D;
  for (int c = tid; c < nk * (D / 8); c += 128) {
    if (!(own && c / (D / 8) == p - c0)) cp_async16(&vs[c / (D / 8)][(c % (D / 8)) * 8], vb + (int64_t)c * 8);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  uint4 kv[D / 8];
  if (tid < nk && !(own && tid == p - c0)) {
    const uint4* kr = reinterpret_cast<const uint4*>(kb + (int64_t)tid * D);
#pragma unroll
    for (int j = 0; j < D / 8; ++j) kv[j] = kr[j];
  }
  if (tid < D / 2) {
    const float c = to_f(cs[(int64_t)p * (D / 2) + tid]), s = to_f(sn[(int64_t)p * (D / 2) + tid]);
    const float q1 = to_f(qkv[hh * D + 2 * tid]), q2 = to_f(qkv[hh * D + 2 * tid + 1]);
    qs[2 * tid] = to_f(Act<T>::from_float(q1 * c - q2 * s));
    qs[2 * tid + 1] = to_f(Act<T>::from_float(q1 * s + q2 * c));
    if (own) {
      const float k1 = to_f(qkv[(H + hh) * D + 2 * tid]), k2 = to_f(qkv[(H + hh) * D + 2 * tid + 1]);
      const T v1 = qkv[(2 * H + hh) * D + 2 * tid], v2 = qkv[(2 * H + hh) * D + 2 * tid + 1];
      const T r1 = Act<T>::from_float(k1 * c - k2 * s), r2 = Act<T>::from_float(k1 * s + k2 * c);
      kp[2 * tid] = r1;
      kp[2 * tid + 1] = r2;
      vs[p - c0][2 * tid] = v1;
      vs[p - c0][2 * tid + 1] = v2;
      T* ko = kc + ((int64_t)hh * S + p) * D;
      ko[2 * tid] = r1;
      ko[2 * tid + 1] = r2;
      T* vo = vc + ((int64_t)hh * S + p) * D;
      vo[2 * tid] = v1;
      vo[2 * tid + 1] = v2;
    }
  }
  __syncthreads();
  float v = -INFINITY;
  if (tid < nk) {
    if (own && tid == p - c0) {
#pragma unroll
      for (int j = 0; j < D / 8; ++j) kv[j] = reinterpret_cast<const uint4*>(kp)[j];
    }
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      float kf[8];
      unpack8<T>(kv[j], kf);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc += qs[8 * j + e] * kf[e];
    }
    v = acc * scale;
  }
  float m = v;
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  const float e = tid < nk ? __expf(v - m) : 0.0f;
  sc[tid] = e;
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  const float z = block_sum(e, red);
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int s0 = warp; s0 < nk; s0 += 4) {
    const uint2 vv = *reinterpret_cast<const uint2*>(&vs[s0][4 * lane]);
    const T* ve = reinterpret_cast<const T*>(&vv);
    const float w = sc[s0];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += w * to_f(ve[q]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) part[warp][4 * lane + q] = acc[q];
  __syncthreads();
  wp[2 + tid] = (part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]);
  if (tid == 0) {
    wp[0] = m;
    wp[1] = z;
  }
}

template <typename T, int D>
__global__ void __launch_bounds__(128) k_attn_combine(const float* __restrict__ ws, const int64_t* __restrict__ pos,
                                                      T* __restrict__ out, int NC, int S) {
  griddep_wait();
  griddep_launch_dependents();
  const int hh = blockIdx.x, tid = threadIdx.x;
  const float* wh = ws + (int64_t)hh * NC * (D + 2);
  if (pos[0] < 0 || pos[0] >= S) {
    out[(int64_t)hh * D + tid] = Act<T>::from_float(0.0f);
    return;
  }
  float M = -INFINITY;
  for (int c = 0; c < NC; ++c) M = fmaxf(M, wh[c * (D + 2)]);
  float L = 0.0f, a = 0.0f;
  for (int c = 0; c < NC; ++c) {   // chunk order: fixed, deterministic
    const float mc = wh[c * (D + 2)];
    if (mc == -INFINITY) continue;
    const float f = __expf(mc - M);
    L += wh[c * (D + 2) + 1] * f;
    a += wh[c * (D + 2) + 2 + tid] * f;
  }
  out[(int64_t)hh * D + tid] = Act<T>::from_float(a / L);
}

// Greedy decode bookkeeping in one kernel (one CTA of 1024 threads): idx = argmax(logits)
// (lowest index among equal maxima), out_tokens[pos] = idx, tok = idx, pos += 1, and the next
// token's embedding row h_next = embed[idx] -- replacing argmax + index_copy + add + the
// embedding gather of the next step (four launches, ~30 us on B200) by one.
template <typename T>
__global__ void __launch_bounds__(1024) k_greedy_next(const T* __restrict__ logits, int vocab,
                                                      int64_t* __restrict__ out_tokens, int max_pos,
                                                      int64_t* __restrict__ tok, int64_t* __restrict__ pos,
                                                      const T* __restrict__ embed, int d, T* __restrict__ h_next) {
  {   // batched decode (tr_greedy_next_batch): sequence blockIdx.x
    const int64_t bq = blockIdx.x;
    logits += bq * vocab;
    out_tokens += bq * max_pos;
    tok += bq;
    pos += bq;
    h_next += bq * d;
  }
  griddep_wait();
  griddep_launch_dependents();
  __shared__ float bv[32];
  __shared__ int bi[32];
  __shared__ int best_idx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  const bool vec = (vocab % 8) == 0 && ((uintptr_t)logits % 16) == 0;
  if (vec) {   // four 16-byte loads in flight before their compares (one L2 round trip, not four)
    for (int i0 = tid * 8; i0 < vocab; i0 += 4 * 1024 * 8) {
      uint4 u[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = i0 + k * 1024 * 8;
        if (i < vocab) u[k] = *reinterpret_cast<const uint4*>(logits + i);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = i0 + k * 1024 * 8;
        if (i >= vocab) break;
        float f[8];
        unpack8<T>(u[k], f);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (f[e] > best) {   // ascending indices per thread: strict > keeps the lowest
            best = f[e];
            idx = i + e;
          }
      }
    }
  } else {
    for (int i = tid; i < vocab; i += 1024) {
      const float f = to_f(logits[i]);
      if (f > best) {
        best = f;
        idx = i;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > best || (ov == best && oi < idx)) {
      best = ov;
      idx = oi;
    }
  }
  if (lane == 0) {
    bv[warp] = best;
    bi[warp] = idx;
  }
  __syncthreads();
  if (warp == 0) {
    best = bv[lane];
    idx = bi[lane];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > best || (ov == best && oi < idx)) {
        best = ov;
        idx = oi;
      }
    }
    if (lane == 0) {
      if (idx >= vocab) idx = 0;   // all -inf / NaN logits
      best_idx = idx;
      const int64_t p = pos[0];
      if (p < max_pos) out_tokens[p] = idx;
      tok[0] = idx;
      pos[0] = p + 1;
    }
  }
  __syncthreads();
  const T* row = embed + (int64_t)best_idx * d;
  for (int j = tid; j < d; j += 1024) h_next[j] = row[j];
}

// gu [T, 2F] = (gate | up) -> out [T, F] = silu(gate) * up   (8 elements per thread)
template <typename T>
__global__ void k_silu_mul(const T* __restrict__ gu, T* __restrict__ out, int F, int64_t n8) {
  griddep_wait();   // PDL: inputs come from the previous kernel
  griddep_launch_dependents();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = (i * 8) / F, f = (i * 8) % F;
    float g[8], u[8], o[8];
    unpack8<T>(*reinterpret_cast<const uint4*>(gu + t * 2 * F + f), g);
    unpack8<T>(*reinterpret_cast<const uint4*>(gu + t * 2 * F + F + f), u);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = to_f(Act<T>::from_float(__fdividef(g[e], 1.0f + __expf(-g[e])))) * u[e];
    *reinterpret_cast<uint4*>(out + t * F + f) = pack8<T>(o);
  }
}

// launch with programmatic dependent launch so chained decode kernels overlap their
// launch latency (the kernels call griddepcontrol.wait before touching their inputs)
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace tr

using namespace tr;

#define TR_ACT_DISPATCH(act, KCALL_H, KCALL_B)                                            \
  do {                                                                                     \
    if ((act) == kActF16) {                                                                \
      KCALL_H;                                                                             \
    } else if ((act) == kActBf16) {                                                        \
      KCALL_B;                                                                             \
    } else {                                                                               \
      TR_REQUIRE(false, "act_dtype must be F16(1) or BF16(2), got %d", (act));            \
    }                                                                                      \
  } while (0)

extern "C" {

int tr_add_rmsnorm(int act, void* h, const void* delta, const void* w, void* y, int64_t rows, int64_t d, float eps,
                   void* stream) {
  TR_REQUIRE(rows >= 0 && d >= 8 && (d % 8) == 0 && d <= 4 * 8 * 1024, "tr_add_rmsnorm: d must be a multiple of 8");
  if (rows == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int nv = (int)(d / 8);
  const int threads = nv <= 1024 ? ((nv + 31) / 32) * 32 : 1024;
  const int V = (int)ceil_div(nv, threads);
  cudaError_t e = cudaSuccess;
#define TR_RMS(TT, VV) e = launch_pdl(k_add_rmsnorm<TT, VV>, dim3((int)rows), dim3(threads), 0, st, (TT*)h, \
                                      (const TT*)delta, (const TT*)w, (TT*)y, (int)d, eps)
  if (act == kActF16) {
    if (V == 1) TR_RMS(__half, 1); else if (V == 2) TR_RMS(__half, 2); else TR_RMS(__half, 4);
  } else if (act == kActBf16) {
    if (V == 1) TR_RMS(__nv_bfloat16, 1); else if (V == 2) TR_RMS(__nv_bfloat16, 2); else TR_RMS(__nv_bfloat16, 4);
  } else {
    TR_REQUIRE(false, "tr_add_rmsnorm: act_dtype must be F16(1) or BF16(2)");
  }
#undef TR_RMS
  (void)e;
  return check_launch("tr_add_rmsnorm");
}

int tr_rope_kv(int act, const void* qkv, const int64_t* pos, const void* cos_t, const void* sin_t, void* q,
               void* k_cache, void* v_cache, int64_t tokens, int64_t heads, int64_t head_dim, int64_t max_seq,
               void* stream) {
  TR_REQUIRE(tokens >= 0 && heads >= 1 && head_dim >= 2 && (head_dim % 2) == 0, "tr_rope_kv: bad shape");
  if (tokens == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)heads, (unsigned)tokens);
  TR_ACT_DISPATCH(act,
                  (launch_pdl(k_rope_kv<__half>, grid, dim3(64), 0, st, (const __half*)qkv, pos, (const __half*)cos_t,
                                                          (const __half*)sin_t, (__half*)q, (__half*)k_cache,
                                                          (__half*)v_cache, (int)heads, (int)head_dim, (int)max_seq)),
                  (launch_pdl(k_rope_kv<__nv_bfloat16>, grid, dim3(64), 0, st, 
                      (const __nv_bfloat16*)qkv, pos, (const __nv_bfloat16*)cos_t, (const __nv_bfloat16*)sin_t,
                      (__nv_bfloat16*)q, (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache, (int)heads,
                      (int)head_dim, (int)max_seq)));
  return check_launch("tr_rope_kv");
}

int tr_attn_decode(int act, const void* qkv, const int64_t* pos, const void* cos_t, const void* sin_t,
                   void* k_cache, void* v_cache, void* out, int64_t heads, int64_t head_dim, int64_t max_seq,
                   float scale, void* stream) {
  TR_REQUIRE(head_dim == 128, "tr_attn_decode: head_dim must be 128");
  TR_REQUIRE(heads >= 1 && max_seq >= 1 && max_seq <= 128, "tr_attn_decode: 1 <= max_seq <= 128");
  cudaStream_t st = (cudaStream_t)stream;
  TR_ACT_DISPATCH(act,
                  (launch_pdl(k_attn_decode<__half, 128>, dim3((int)heads), dim3(128), 0, st, (const __half*)qkv,
                              pos, (const __half*)cos_t, (const __half*)sin_t, (__half*)k_cache, (__half*)v_cache,
                              (__half*)out, (int)heads, (int)max_seq, scale)),
                  (launch_pdl(k_attn_decode<__nv_bfloat16, 128>, dim3((int)heads), dim3(128), 0, st,
                              (const __nv_bfloat16*)qkv, pos, (const __nv_bfloat16*)cos_t,
                              (const __nv_bfloat16*)sin_t, (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache,
                              (__nv_bfloat16*)out, (int)heads, (int)max_seq, scale)));
  return check_launch("tr_attn_decode");
}

size_t tr_attn_decode_workspace_size(int64_t heads, int64_t head_dim, int64_t max_seq) {
  if (heads < 1 || head_dim != 128 || max_seq < 1) return 0;
  return (size_t)heads * ceil_div(max_seq, 128) * (head_dim + 2) * sizeof(float);
}

int tr_attn_decode_split(int act, const void* qkv, const int64_t* pos, const void* cos_t, const void* sin_t,
                         void* k_cache, void* v_cache, void* out, int64_t heads, int64_t head_dim, int64_t max_seq,
                         float scale, void* workspace, size_t ws_bytes, void* stream) {
  TR_REQUIRE(head_dim == 128, "tr_attn_decode_split: head_dim must be 128");
  TR_REQUIRE(heads >= 1 && max_seq >= 1 && max_seq < (1LL << 24), "tr_attn_decode_split: bad heads / max_seq");
  TR_REQUIRE(workspace && ws_bytes >= tr_attn_decode_workspace_size(heads, head_dim, max_seq),
             "tr_attn_decode_split: workspace too small (tr_attn_decode_workspace_size)");
  cudaStream_t st = (cudaStream_t)stream;
  const int nc = (int)ceil_div(max_seq, 128);
  float* ws = (float*)workspace;
  TR_ACT_DISPATCH(act,
                  (launch_pdl(k_attn_split<__half, 128>, dim3((int)heads, nc), dim3(128), 0, st, (const __half*)qkv,
                              pos, (const __half*)cos_t, (const __half*)sin_t, (__half*)k_cache, (__half*)v_cache, ws,
                              (int)heads, (int)max_seq, scale)),
                  (launch_pdl(k_attn_split<__nv_bfloat16, 128>, dim3((int)heads, nc), dim3(128), 0, st,
                              (const __nv_bfloat16*)qkv, pos, (const __nv_bfloat16*)cos_t,
                              (const __nv_bfloat16*)sin_t, (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache, ws,
                              (int)heads, (int)max_seq, scale)));
  if (check_launch("tr_attn_decode_split")) return -1;
  TR_ACT_DISPATCH(act,
                  (launch_pdl(k_attn_combine<__half, 128>, dim3((int)heads), dim3(128), 0, st, (const float*)ws, pos,
                              (__half*)out, nc, (int)max_seq)),
                  (launch_pdl(k_attn_combine<__nv_bfloat16, 128>, dim3((int)heads), dim3(128), 0, st,
                              (const float*)ws, pos, (__nv_bfloat16*)out, nc, (int)max_seq)));
  return check_launch("tr_attn_decode_split(combine)");
}

int tr_silu_mul(int act, const void* gu, void* out, int64_t tokens, int64_t ff, void* stream) {
  TR_REQUIRE(tokens >= 0 && ff >= 8 && (ff % 8) == 0, "tr_silu_mul: ff must be a multiple of 8");
  const int64_t n8 = tokens * ff / 8;
  if (n8 == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)(ceil_div(n8, 256) > 148 * 8 ? 148 * 8 : ceil_div(n8, 256));
  TR_ACT_DISPATCH(act,
                  (launch_pdl(k_silu_mul<__half>, dim3(grid), dim3(256), 0, st, (const __half*)gu, (__half*)out,
                              (int)ff, n8)),
                  (launch_pdl(k_silu_mul<__nv_bfloat16>, dim3(grid), dim3(256), 0, st, (const __nv_bfloat16*)gu,
                              (__nv_bfloat16*)out, (int)ff, n8)));
  return check_launch("tr_silu_mul");
}

int tr_attn_decode_batch(int act, const void* qkv, const int64_t* pos, const void* cos_t, const void* sin_t,
                         void* k_cache, void* v_cache, void* out, int64_t batch, int64_t heads, int64_t head_dim,
                         int64_t max_seq, float scale, void* stream) {
  TR_REQUIRE(head_dim == 128, "tr_attn_decode_batch: head_dim must be 128");
  TR_REQUIRE(heads >= 1 && max_seq >= 1 && max_seq <= 128, "tr_attn_decode_batch: 1 <= max_seq <= 128");
  TR_REQUIRE(batch >= 1 && batch <= 65535, "tr_attn_decode_batch: 1 <= batch <= 65535");
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((unsigned)heads, (unsigned)batch);
  TR_ACT_DISPATCH(act,
                  (launch_pdl(k_attn_decode<__half, 128>, grid, dim3(128), 0, st, (const __half*)qkv, pos,
                              (const __half*)cos_t, (const __half*)sin_t, (__half*)k_cache, (__half*)v_cache,
                              (__half*)out, (int)heads, (int)max_seq, scale)),
                  (launch_pdl(k_attn_decode<__nv_bfloat16, 128>, grid, dim3(128), 0, st, (const __nv_bfloat16*)qkv,
                              pos, (const __nv_bfloat16*)cos_t, (const __nv_bfloat16*)sin_t,
                              (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache, (__nv_bfloat16*)out, (int)heads,
                              (int)max_seq, scale)));
  return check_launch("tr_attn_decode_batch");
}
int tr_greedy_next_batch(int act, const void* logits, int64_t vocab, int64_t* out_tokens, int64_t max_pos,
                         int64_t* tok, int64_t* pos, const void* embed, int64_t d, void* h_next, int64_t batch,
                         void* stream) {
  TR_REQUIRE(vocab >= 1 && vocab < (1LL << 31) && d >= 1 && max_pos >= 0, "tr_greedy_next_batch: bad sizes");
  TR_REQUIRE(batch >= 1 && batch <= 65535, "tr_greedy_next_batch: 1 <= batch <= 65535");
  cudaStream_t st = (cudaStream_t)stream;
  TR_ACT_DISPATCH(act,
                  (launch_pdl(k_greedy_next<__half>, dim3((unsigned)batch), dim3(1024), 0, st, (const __half*)logits,
                              (int)vocab, out_tokens, (int)max_pos, tok, pos, (const __half*)embed, (int)d,
                              (__half*)h_next)),
                  (launch_pdl(k_greedy_next<__nv_bfloat16>, dim3((unsigned)batch), dim3(1024), 0, st,
                              (const __nv_bfloat16*)logits, (int)vocab, out_tokens, (int)max_pos, tok, pos,
                              (const __nv_bfloat16*)embed, (int)d, (__nv_bfloat16*)h_next)));
  return check_launch("tr_greedy_next_batch");
}
int tr_greedy_next(int act, const void* logits, int64_t vocab, int64_t* out_tokens, int64_t max_pos, int64_t* tok,
                   int64_t* pos, const void* embed, int64_t d, void* h_next, void* stream) {
  TR_REQUIRE(vocab >= 1 && vocab < (1LL << 31) && d >= 1 && max_pos >= 0, "tr_greedy_next: bad sizes");
  cudaStream_t st = (cudaStream_t)stream;
  TR_ACT_DISPATCH(act,
                  (launch_pdl(k_greedy_next<__half>, dim3(1), dim3(1024), 0, st, (const __half*)logits, (int)vocab,
                              out_tokens, (int)max_pos, tok, pos, (const __half*)embed, (int)d, (__half*)h_next)),
                  (launch_pdl(k_greedy_next<__nv_bfloat16>, dim3(1), dim3(1024), 0, st, (const __nv_bfloat16*)logits,
                              (int)vocab, out_tokens, (int)max_pos, tok, pos, (const __nv_bfloat16*)embed, (int)d,
                              (__nv_bfloat16*)h_next)));
  return check_launch("tr_greedy_next");
}

}  // extern "C"
