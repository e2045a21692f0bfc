// Single-token decode attention for one head, run by one 128-thread group of a larger CTA
// (thread index tid 0..127, its own named barrier): the body of k_attn_decode (decode_ops.cu) as a device function, so the fused
// QKV-GEMV + attention kernel (gemv_s8.cu, ATT = 1) can finish a head inside the cluster that
// produced its q / k / v rows.  Same arithmetic and roundings as k_attn_decode:
//   q, k rotated (rotary angle table cs / sn [S, D/2]) and rounded to T; k, v appended to the
//   caches [H, S, D] at pos; out[hh] = softmax(q k^T * scale over keys 0..pos) v, fp32 sums.
#pragma once

#include "common.cuh"

namespace tr {

namespace attn {

template <typename T> __device__ __forceinline__ float tof(T v);
template <> __device__ __forceinline__ float tof<__half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float tof<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ void bar128(int id) { asm volatile("bar.sync %0, 128;\n" ::"r"(id) : "memory"); }

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// bytes of shared memory attn_head_128 needs at `sm` (16-byte aligned)
constexpr int kSmemBytes = 128 * 128 * 2 + 128 * 2 + (128 + 128 + 4 * 128 + 32) * 4;

__device__ __forceinline__ float sum128(float v, float* red, int tid, int bar) {   // one group, fixed order
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = tid >> 5, lane = tid & 31;
  bar128(bar);
  if (lane == 0) red[warp] = v;
  bar128(bar);
  return ((red[0] + red[1]) + red[2]) + red[3];   // (k_attn_decode's block_sum order)
}

// qkv: [3, H, D] of this token (written by other CTAs of the cluster: read through L2).
template <typename T>
__device__ void attn_head_128(const T* qkv, const int64_t* pos, const T* cs, const T* sn, T* kc, T* vc, T* out,
                              int H, int S, int hh, float scale, uint8_t* sm, int tid, int bar) {
  constexpr int D = 128;
  T (*vs)[D] = reinterpret_cast<T (*)[D]>(sm);
  T* kp = reinterpret_cast<T*>(sm + 128 * D * sizeof(T));
  float* qs = reinterpret_cast<float*>(kp + D);
  float* sc = qs + D;
  float* part = sc + 128;
  float* red = part + 4 * D;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t p64 = pos[0];
  if (p64 < 0 || p64 >= S) {   // past the cache: write nothing into it, output zeros
    out[(int64_t)hh * D + tid] = Act<T>::from_float(0.0f);
    return;
  }
  const int p = (int)p64, n = p + 1;
  const T* kb = kc + (int64_t)hh * S * D;
  const T* vb = vc + (int64_t)hh * S * D;
  for (int c = tid; c < p * (D / 8); c += 128) cp_async16(&vs[c / (D / 8)][(c % (D / 8)) * 8], vb + (int64_t)c * 8);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  uint4 kv[D / 8];
  if (tid < p) {
    const uint4* kr = reinterpret_cast<const uint4*>(kb + (int64_t)tid * D);
#pragma unroll
    for (int j = 0; j < D / 8; ++j) kv[j] = kr[j];
  }
  if (tid < D / 2) {
    const float c = tof(cs[(int64_t)p * (D / 2) + tid]), s = tof(sn[(int64_t)p * (D / 2) + tid]);
    const float q1 = tof(__ldcg(qkv + hh * D + 2 * tid)), q2 = tof(__ldcg(qkv + hh * D + 2 * tid + 1));
    const float k1 = tof(__ldcg(qkv + (H + hh) * D + 2 * tid)), k2 = tof(__ldcg(qkv + (H + hh) * D + 2 * tid + 1));
    const T v1 = __ldcg(qkv + (2 * H + hh) * D + 2 * tid), v2 = __ldcg(qkv + (2 * H + hh) * D + 2 * tid + 1);
    qs[2 * tid] = tof(Act<T>::from_float(q1 * c - q2 * s));
    qs[2 * tid + 1] = tof(Act<T>::from_float(q1 * s + q2 * c));
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
  bar128(bar);
  float v = -INFINITY;
  if (tid <= p) {
    if (tid == p) {
#pragma unroll
      for (int j = 0; j < D / 8; ++j) kv[j] = reinterpret_cast<const uint4*>(kp)[j];
    }
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      const T* e8 = reinterpret_cast<const T*>(&kv[j]);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc += qs[8 * j + e] * tof(e8[e]);
    }
    v = acc * scale;
  }
  float m = v;
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[8 + warp] = m;
  bar128(bar);
  m = fmaxf(fmaxf(red[8], red[9]), fmaxf(red[10], red[11]));
  const float e = tid < n ? __expf(v - m) : 0.0f;
  sc[tid] = e;
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");   // (sum128 syncs: values visible after it)
  const float z = sum128(e, red, tid, bar);
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int s0 = warp; s0 < n; s0 += 4) {
    const uint2 vv = *reinterpret_cast<const uint2*>(&vs[s0][4 * lane]);
    const T* ve = reinterpret_cast<const T*>(&vv);
    const float w = sc[s0];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += w * tof(ve[q]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) part[warp * D + 4 * lane + q] = acc[q];
  bar128(bar);
  const float r = ((part[tid] + part[D + tid]) + (part[2 * D + tid] + part[3 * D + tid])) / z;
  out[(int64_t)hh * D + tid] = Act<T>::from_float(r);
}

}  // namespace attn
}  // namespace tr
