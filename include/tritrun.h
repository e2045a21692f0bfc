/*
 * tritrun.h -- C-ABI of libtritrun.so, the B200 (sm_100a) TriRun hot path.
 *
 * Drop-in boundary for the reference package `tritpack`
 * (/root/reference/pkg/src/tritpack).  The reference plugs kernels in through
 * backend.resolve() (backend.py:54-63), which returns a *kernel module* with the
 * duck-typed surface of _kernels.pyx:23-227 / _kernels_py.py:46-171.  Every
 * entry point below is either one function of that surface (same argument
 * meaning, same bit-exact results) or a piece of the GPU path the paper's
 * TriRun kernel adds (repacker, fp16/bf16 GEMV/GEMM, dense dequant).
 *
 * Conventions:
 *   - all array arguments are DEVICE pointers owned by the caller; nothing is
 *     allocated on the hot path and nothing synchronises the host;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); every call is
 *     stream-ordered and thread-safe;
 *   - return 0 on success, -1 on a rejected argument or CUDA launch error, with
 *     a message in tr_last_error() (per calling thread).  The reference kernels
 *     do no validation (_kernels.pyx:2-4); its Python callers raise ValueError
 *     (linear.py:104-108, 123-129), which the Python host layer mirrors.
 *   - fmt uses the reference DType tags: TQ2 = 2, TQ1 = 3 (blocks.py:45-52).
 *   - act_dtype: 1 = fp16, 2 = bf16.
 */
#ifndef TRITRUN_H
#define TRITRUN_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TR_API __attribute__((visibility("default")))
#else
#define TR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define TR_FMT_TQ2 2
#define TR_FMT_TQ1 3
#define TR_ACT_F16 1
#define TR_ACT_BF16 2
#define TR_LINEAR_PDL 1            /* flags bit 0: launch with programmatic dependent launch */
#define TR_LINEAR_UNIFORM_SCALE 2  /* bit 1: caller asserts each row has one scale for all its blocks */
#define TR_LINEAR_FORCE_UMMA 4     /* bit 2: force the tcgen05 tensor-core GEMM */
#define TR_LINEAR_FORCE_GEMV 8     /* bit 3: force the mma.sync GEMV */
#define TR_LINEAR_GEMV_F16 16      /* bit 4: batch 1-4 on the fp16 GEMV instead of the int8-slice one */
#define TR_LINEAR_COSCHEDULE 32    /* bit 5: chained with other GEMVs back to back: run the int8-slice GEMV
                                    * as 8-warp (half-SM) CTAs, so a layer and its successor can share
                                    * SMs (the successor prefetches its weights early); measured +5%
                                    * on the BASELINE layer stack, neutral-to-worse as a default;
                                    * batch 1 only: batch >= 2 always runs 16 warps */
#define TR_LINEAR_FULL_SM (1 << 28) /* bit 28: the int8-slice GEMV as 16-warp (whole-SM) CTAs at batch 1
                                    * too (the decoder's fused-attention step measures best with it) */
#define TR_LINEAR_EPI_SWIGLU 64    /* bit 6: W's rows are 16-row tiles alternating gate / up (2 F rows);
                                    * y[batch, F] = silu(gate) * up with the roundings of an fp16/bf16
                                    * gate|up store followed by tr_silu_mul (int8-slice GEMV at batch
                                    * <= 4, or the tcgen05 GEMM where the dispatch picks it: rows a
                                    * multiple of 32, 16-byte aligned activation rows) */
#define TR_LINEAR_OUT_F32 128      /* bit 7: y is float32 (the fp32 accumulators, not rounded to the
                                    * activation type): row-parallel partials for an fp32 all-reduce */

TR_API const char* tr_last_error(void);
TR_API int tr_version(void);

/* ---- reference kernel-module surface (bit-exact) --------------------------- */

/* _kernels.pyx:23-35 pack_base4: digits u8[4m] -> words u8[m] */
TR_API int tr_pack_base4(const uint8_t* digits, uint8_t* words, int64_t m, void* stream);
/* _kernels.pyx:38-52 unpack_base4: words u8[m] -> digits u8[4m] */
TR_API int tr_unpack_base4(const uint8_t* words, uint8_t* digits, int64_t m, void* stream);
/* _kernels.pyx:55-70 encode_base3: digits u8[5m] -> codes u8[m] */
TR_API int tr_encode_base3(const uint8_t* digits, uint8_t* codes, int64_t m, void* stream);
/* _kernels.pyx:73-87 decode_base3 (Algorithm 1): codes u8[m] -> digits u8[5m] */
TR_API int tr_decode_base3(const uint8_t* codes, uint8_t* digits, int64_t m, void* stream);
/* _kernels.pyx:90-118 quantize_blocks: f32[nb,256] -> digits u8[nb,256], absmax f32[nb] */
TR_API int tr_quantize_blocks(const float* values, uint8_t* digits, float* scales, int64_t nb, void* stream);
/* _kernels.pyx:121-133 dequantize_blocks: digits u8[nb,256], f32[nb] -> f32[nb,256] */
TR_API int tr_dequantize_blocks(const uint8_t* digits, const float* scales, float* out, int64_t nb,
                                void* stream);
/* _kernels.pyx:171-227 gemm_tq2 / gemm_tq1, bit-exact parity mode:
 * payload u8[rows,nb,64|52], scales f32[rows,nb], x f32[batch, nb*256] (zero-padded
 * by the caller, linear.py:151-152), out f32[batch,rows]; columns [row0,row1) written. */
TR_API int tr_gemm_exact(int fmt, const uint8_t* payload, const float* scales, const float* x, float* out,
                         int64_t rows, int64_t nb, int64_t batch, int64_t row0, int64_t row1, void* stream);

/* ---- offline packing / repacking ------------------------------------------------ */

/* linear.py:98-120 pack_matrix (+ blocks.py:142-161 quantize_rows) on the device:
 * W f32[rows,cols] -> payload u8[rows,nb,64|52] + binary16 scales u16[rows,nb]. */
TR_API int tr_quantize_pack(int fmt, const float* W, int64_t rows, int64_t cols, uint8_t* payload,
                            uint16_t* scales_f16, void* stream);
/* bytes of the device ("T16") layout of a rows x cols matrix (-1 if unsupported) */
TR_API int64_t tr_layout_bytes(int fmt, int64_t rows, int64_t cols);
/* PackedMatrix (linear.py:29-95: payload + scales) -> device layout; bit-exactly invertible.
 * dst_bytes: the size of dst (>= tr_layout_bytes(fmt, rows, cols), else -1 and nothing is written) */
TR_API int tr_repack(int fmt, const uint8_t* payload, const uint16_t* scales_f16, int64_t rows, int64_t cols,
                     void* dst, size_t dst_bytes, void* stream);
/* device layout -> PackedMatrix payload + scales (exact inverse of tr_repack) */
/* TPK1 container (container.py:73-82, 167-242) -> device tiles in one pass: records = the
 * data section of one TQ2/TQ1 tensor on the device, rows x ceil(cols/256) records of
 * payload (64|52 B) followed by its binary16 scale (66|54 B each, no padding). */
TR_API int tr_repack_records(int fmt, const uint8_t* records, int64_t rows, int64_t cols, void* dst,
                             size_t dst_bytes, void* stream);
TR_API int tr_unrepack(int fmt, const void* src, int64_t rows, int64_t cols, size_t src_bytes, uint8_t* payload,
                       uint16_t* scales_f16, void* stream);
/* linear.py:177-198 dequantize_matrix, to a dense fp16/bf16 [rows, cols] matrix
 * (values scale*(d-1) are exact in fp16); feeds the cuBLAS baseline. */
TR_API int tr_dequant_dense(int fmt, const uint8_t* payload, const uint16_t* scales_f16, int64_t rows,
                            int64_t cols, int act_dtype, void* out, void* stream);

/* ---- the hot path ------------------------------------------------------------------ */

/* Bytes of caller-owned device workspace tr_linear needs for this shape (0 on bad
 * arguments).  The first 256 KiB are per-tile arrival counters: ZERO them once
 * after allocating; kernels leave them zeroed.  One workspace per stream. */
TR_API size_t tr_linear_workspace_size(int fmt, int64_t batch, int64_t rows, int64_t cols);
/* y[batch, rows] = x[batch, cols] @ W^T  (linear.py:137-166 gemm semantics with the
 * paper's fp16/bf16 activations, fp32 accumulation, RNE output).  w is the device
 * layout from tr_repack; x has leading dimension ldx, y has ldy (elements).
 * Dispatch (measured crossovers): batch 1-2 run the int8-slice GEMV (K3-S8:
 * exact integer block sums over activations put on a 2^-24 grid of each 256-column block's
 * maximum; TQ1 weights: K4), except batch 2 with more than 8192 columns spread over <= 8
 * blocks per GEMM CTA; everything else the tcgen05 GEMM (K5).  The fp16 mma.sync GEMV (K3) runs on request (TR_LINEAR_GEMV_F16 / FORCE_GEMV) and
 * where K3-S8 cannot stage the activations and K5 cannot take them (unaligned rows).
 * flags: TR_LINEAR_* bits | (knob << 8): GEMV CTA count / GEMM K split (0 = automatic). */
TR_API int tr_linear(int fmt, const void* w, const void* x, void* y, int64_t batch, int64_t rows, int64_t cols,
                     int act_dtype, int64_t ldx, int64_t ldy, int flags, void* workspace, size_t ws_bytes,
                     void* stream);

/* tr_linear with the producer of x fused into the GEMV's activation staging (decode glue;
 * batch 1..8, TQ2, activations that fit in shared memory -- else -1):
 *  TR_PRE_ADD_RMSNORM: x_eff = rmsnorm(x + delta) * gamma (delta may be NULL); x + delta
 *     (rounded) is also stored to x_out [batch, cols] (stride ldx) -- must not alias x;
 *  TR_PRE_SILU_MUL:    x_eff = silu(x[:, :cols]) * x[:, cols:2 cols]  (x = gate|up, ldx >= 2 cols).
 * Same arithmetic and roundings as tr_add_rmsnorm / tr_silu_mul followed by tr_linear.
 * Under TR_LINEAR_PDL, w and gamma are read before the launch waits on the previous kernel
 * (parameters, not activations): they must not be written by the kernel just before. */
#define TR_PRE_ADD_RMSNORM 1
#define TR_PRE_SILU_MUL 2
TR_API int tr_linear_pre(int fmt, const void* w, const void* x, void* y, int64_t batch, int64_t rows, int64_t cols,
                         int act_dtype, int64_t ldx, int64_t ldy, int flags, int pre_op, const void* delta,
                         const void* gamma, void* x_out, float eps, void* stream);

/* One product of a chain (tr_linear_chain): y[batch, rows] = x_eff[batch, cols] @ W^T, TQ2 device
 * layout, where x_eff is x or, with pre_op, its fused producer exactly as in tr_linear_pre
 * (TR_PRE_ADD_RMSNORM: rmsnorm(x + delta) * gamma, x + delta stored to x_out; TR_PRE_SILU_MUL:
 * silu(x[:, :cols]) * x[:, cols:]).  flags: TR_LINEAR_EPI_SWIGLU (rows are gate/up tile pairs,
 * y is rows/2 wide) or TR_LINEAR_OUT_F32. */
typedef struct {
  const void* w;
  const void* x;
  void* y;
  int64_t ldx, ldy, rows, cols;
  int32_t pre_op;        /* 0, TR_PRE_ADD_RMSNORM or TR_PRE_SILU_MUL */
  int32_t flags;         /* TR_LINEAR_EPI_SWIGLU | TR_LINEAR_OUT_F32 */
  const void* delta;     /* TR_PRE_ADD_RMSNORM: added to x (may be NULL) */
  const void* gamma;     /* TR_PRE_ADD_RMSNORM: norm weight [cols] */
  void* x_out;           /* TR_PRE_ADD_RMSNORM: receives x + delta (may be NULL) */
  float eps;
} TrChainLayer;

/* Bytes of caller-owned device workspace tr_linear_chain needs for n_layers (zero it once: the
 * first 4 KiB hold the per-product arrival counters, which every launch leaves zeroed). */
TR_API size_t tr_linear_chain_workspace_size(int64_t n_layers);
/* Validate the chain and upload its product table into the workspace (synchronous; call once,
 * outside any stream capture, and again whenever a pointer or shape changes). */
TR_API int tr_linear_chain_prepare(const TrChainLayer* layers, int64_t n_layers, int64_t batch, void* workspace,
                                   size_t ws_bytes);
/* A dependent chain of products (layer l reads what layers < l wrote) for batch 1..4 in ONE
 * persistent launch (K6): one CTA per SM, each warp's TMA weight ring streaming the next
 * products' weights while the grid waits for a product's inputs; products ordered by arrival
 * counters in the workspace, not kernel boundaries.  Same arithmetic as tr_linear /
 * tr_linear_pre on the int8-slice GEMV.  `layers` is the HOST array given to
 * tr_linear_chain_prepare; graph-capturable.  (up to 256 products) */
TR_API int tr_linear_chain(int act_dtype, const TrChainLayer* layers, int64_t n_layers, int64_t batch, int flags,
                           void* workspace, size_t ws_bytes, void* stream);

/* ---- decoder-layer glue (configs[2] decode stack; no reference analogue) ---------- */

/* One decode token's attention block input side in ONE kernel: x = rmsnorm(h + delta) * gamma (h + delta
 * stored to h_out), qkv_out [3, H, D] = x W_qkv^T (TQ2 device layout, rows 3 H D, cols H D), then
 * tr_attn_decode on qkv_out (rotary, cache append at pos[0], softmax attention) -> att_out [H, D].
 * Six CTAs share each head's 24 tiles; the last to finish runs the head's attention.  Same
 * roundings as tr_linear_pre + tr_attn_decode.  head_dim 128, max_seq <= 128, batch 1.
 * workspace: tr_qkv_attn_decode_workspace_size(heads) bytes of per-head arrival counters, zeroed
 * once by the caller; every launch leaves them zero again (one launch in flight per workspace). */
TR_API size_t tr_qkv_attn_decode_workspace_size(int64_t heads);
TR_API int tr_qkv_attn_decode(int act_dtype, const void* w_qkv, const void* h, const void* delta, const void* gamma,
                              void* h_out, float eps, void* qkv_out, const int64_t* pos, const void* cos_t,
                              const void* sin_t, void* k_cache, void* v_cache, void* att_out, int64_t heads,
                              int64_t head_dim, int64_t max_seq, float scale, void* workspace, size_t ws_bytes,
                              int flags, void* stream);

/* h[r] += delta[r] (delta may be NULL); y[r] = h[r] * rsqrt(mean(h[r]^2) + eps) * w; rows x d */
TR_API int tr_add_rmsnorm(int act_dtype, void* h, const void* delta, const void* w, void* y, int64_t rows,
                          int64_t d, float eps, void* stream);
/* qkv [T,3,H,D] -> rotary q [T,H,D]; rotary k and v appended to k/v caches [H,S,D] at pos[t] (int64, device) */
TR_API int tr_rope_kv(int act_dtype, const void* qkv, const int64_t* pos, const void* cos_t, const void* sin_t,
                      void* q, void* k_cache, void* v_cache, int64_t tokens, int64_t heads, int64_t head_dim,
                      int64_t max_seq, void* stream);
/* one decode token, fused: rotary q/k of qkv [3,H,D] at pos[0], k/v appended to the caches
 * [H,S,D], out [H,D] = softmax(q k^T scale over keys 0..pos[0]) v  (head_dim 128, S <= 128) */
TR_API int tr_attn_decode(int act_dtype, const void* qkv, const int64_t* pos, const void* cos_t, const void* sin_t,
                          void* k_cache, void* v_cache, void* out, int64_t heads, int64_t head_dim, int64_t max_seq,
                          float scale, void* stream);
/* tr_attn_decode for any cache length (split-KV: 128 keys per CTA, partial softmaxes merged in a
 * second kernel); workspace: tr_attn_decode_workspace_size bytes of device memory (no init needed) */
TR_API size_t tr_attn_decode_workspace_size(int64_t heads, int64_t head_dim, int64_t max_seq);
TR_API int tr_attn_decode_split(int act_dtype, const void* qkv, const int64_t* pos, const void* cos_t,
                                const void* sin_t, void* k_cache, void* v_cache, void* out, int64_t heads,
                                int64_t head_dim, int64_t max_seq, float scale, void* workspace, size_t ws_bytes,
                                void* stream);
/* gu [T, 2F] = (gate | up) -> out [T, F] = silu(gate) * up */
TR_API int tr_silu_mul(int act_dtype, const void* gu, void* out, int64_t tokens, int64_t ff, void* stream);
/* greedy decode step: idx = argmax(logits [vocab]) (lowest index among ties); out_tokens[pos[0]] = idx
 * (if pos[0] < max_pos); tok[0] = idx; pos[0] += 1; h_next [d] = embed [vocab, d] row idx.  int64 on device. */
TR_API int tr_greedy_next(int act_dtype, const void* logits, int64_t vocab, int64_t* out_tokens, int64_t max_pos,
                          int64_t* tok, int64_t* pos, const void* embed, int64_t d, void* h_next, void* stream);
/* Batched decode (B independent sequences, one token each): the same kernels over a batch of
 * sequences.  tr_attn_decode_batch: qkv [B, 3, H, D], pos [B], caches [B, H, S, D], out [B, H, D].
 * tr_greedy_next_batch: logits [B, vocab], out_tokens [B, max_pos], tok [B], pos [B], h_next [B, d]. */
TR_API int tr_attn_decode_batch(int act_dtype, const void* qkv, const int64_t* pos, const void* cos_t,
                                const void* sin_t, void* k_cache, void* v_cache, void* out, int64_t batch,
                                int64_t heads, int64_t head_dim, int64_t max_seq, float scale, void* stream);
TR_API int tr_greedy_next_batch(int act_dtype, const void* logits, int64_t vocab, int64_t* out_tokens,
                                int64_t max_pos, int64_t* tok, int64_t* pos, const void* embed, int64_t d,
                                void* h_next, int64_t batch, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TRITRUN_H */
