// C-ABI entry points of libtritrun.so (declared in include/tritrun.h) that are
// not defined next to their kernels: error plumbing, version, and the hot-path
// dispatcher tr_linear (decoder-layer linear dispatch: GEMV / skinny-GEMM by
// batch).
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace tr {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: CUDA error: %s", what, cudaGetErrorString(e));
    return -1;
  }
  return 0;
}

int gemv_tq2(int act, const void* w, const void* x, void* y, int64_t ldx, int64_t ldy, int batch, int rows,
             int cols, int ctas, int pdl, cudaStream_t st, int pre, const void* pre_delta, const void* pre_gamma,
             void* pre_out, float eps, int out_f32);
size_t gemv_workspace_bytes(int batch, int rows, int cols);
bool gemv_s8_fits(int batch, int rows, int cols, int fmt);
int gemv_s8(int act, const void* w, const void* x, void* y, int64_t ldx, int64_t ldy, int batch, int rows, int cols,
            int ctas, int pdl, cudaStream_t st, int pre, const void* pre_delta, const void* pre_gamma, void* pre_out,
            float eps, int cosched, int epi, int out_f32, int fmt);
int gemm_umma(int fmt, int act, const void* w, const void* x, void* y, int64_t ldx, int64_t ldy, int batch, int rows,
              int cols, int ks, int uniform, void* workspace, size_t ws_bytes, int pdl, cudaStream_t st, int dbg,
              int out_f32, int epi);
size_t umma_workspace_bytes(int batch, int rows, int cols);
int umma_blocks_per_cta(int batch, int rows, int cols);
int gemv_qkv_attn(int act, const void* w, const void* h, const void* delta, const void* gamma, void* h_out,
                  float eps, void* qkv, const int64_t* pos, const void* cos_t, const void* sin_t, void* k_cache,
                  void* v_cache, void* att_out, int heads, int head_dim, int max_seq, float scale, void* counters,
                  int pdl, int dbg, cudaStream_t st);
bool gemv_stages_x(int batch, int rows, int cols);
int gemv_chain_s8(int act, const TrChainLayer* host, int n, int batch, void* ws, size_t ws_bytes, int flags,
                  cudaStream_t st, bool upload);
size_t chain_workspace_bytes(int n_ops);

// GEMV / tensor-core GEMM crossover, measured per shape at batch 2-12 (scripts/dev/crossover.py,
// then in the BASELINE stack and the batched decoder; DESIGN.md section 4 "Dispatch"): the GEMVs
// restage every activation row in every CTA, so their cost grows with batch x cols; K5 costs about
// the same for any batch up to 16 but pays a fixed cost per CTA and spreads poorly when a shape has
// few 128-row tiles.
//  * batch 1: the int8-slice GEMV (TQ2) / K4 (TQ1);
//  * batch 2: the same, except K > 8192 columns spread over <= 8 blocks per K5 CTA (3072 x 9216);
//  * batch >= 3: K5 (the fp16 GEMV K3 only for activation rows K5 cannot take).
// int8-slice GEMV CTA width: 1 = half-SM 8-warp CTAs (TR_LINEAR_COSCHEDULE), 2 = whole-SM 16-warp
// CTAs (TR_LINEAR_FULL_SM), 0 = by shape
static int sched_mode(int flags) {
  return (flags & TR_LINEAR_FULL_SM) ? 2 : (flags & TR_LINEAR_COSCHEDULE) ? 1 : 0;
}
#ifndef TR_B34_UMMA_ALL
#define TR_B34_UMMA_ALL 1
#endif
static bool prefer_umma(int64_t batch, int64_t rows, int64_t cols) {
  if (batch == 1) return false;
  // blocks each K5 CTA walks: how well the GEMM spreads this shape
  const int bpc = umma_blocks_per_cta((int)batch, (int)rows, (int)cols);
  // batch 2: K5 for long K spread thin (after K5's interleaved decode and 4-stage weight ring at
  // N = 16; scripts/dev/crossover.py: 3072x9216 (6 blocks per CTA) K5 7.51 vs GEMV 8.27 us, batched
  // 3.9B decode B=2 1858 -> 1990 tok/s; 4096x11008 (11 blocks) 8.68 vs 8.81 isolated but 6% slower in
  // the BASELINE stack, so it stays on the GEMV)
  if (batch == 2) return cols > 8192 && bpc <= 8;
  // batch 3-4: K5 everywhere (11008x4096 b=4 8.52 vs 8.64, 4096^2 6.03 vs 6.69; BASELINE stack b=3-4
  // 0.785 -> 0.751 ms; the one shape the GEMV still wins, 9216x3072, by 1.2%)
  if (TR_B34_UMMA_ALL && batch <= 4) return true;
  // (before those changes: 4096^2 b=3-4 K5 6.0-6.1 vs GEMV 6.7 us; 9216x3072 b=4 GEMV 7.6 vs 8.0;
  // 11008x4096 b=4 GEMV 8.5 vs 9.5; from b=5 K5 wins every shape)
  if (batch <= 4) return cols > 8192 || (cols > 4096 && bpc < 12) || bpc <= 4;
  return true;
}
}  // namespace tr

using namespace tr;

extern "C" {

const char* tr_last_error(void) { return g_err; }

int tr_version(void) { return 1; }

size_t tr_linear_workspace_size(int fmt, int64_t batch, int64_t rows, int64_t cols) {
  if ((fmt != kFmtTq2 && fmt != kFmtTq1) || rows < 1 || cols < 1 || batch < 0) return 0;
  const size_t g = 256 * 1024 + gemv_workspace_bytes((int)(batch < 32 ? batch : 32), (int)rows, (int)cols);
  const size_t u = umma_workspace_bytes((int)(batch > 0 ? batch : 1), (int)rows, (int)cols);
  return g > u ? g : u;
}

int tr_linear(int fmt, const void* w, const void* x, void* y, int64_t batch, int64_t rows, int64_t cols,
              int act_dtype, int64_t ldx, int64_t ldy, int flags, void* workspace, size_t ws_bytes,
              void* stream) {
  TR_REQUIRE(fmt == kFmtTq2 || fmt == kFmtTq1, "tr_linear: fmt must be TQ2 (2) or TQ1 (3), got %d", fmt);
  TR_REQUIRE(act_dtype == kActF16 || act_dtype == kActBf16, "tr_linear: act_dtype must be F16(1) or BF16(2)");
  TR_REQUIRE(rows >= 1 && cols >= 1 && batch >= 0, "tr_linear: bad shape batch=%lld rows=%lld cols=%lld",
             (long long)batch, (long long)rows, (long long)cols);
  TR_REQUIRE(rows < (1LL << 30) && cols < (1LL << 30), "tr_linear: shape too large");
  TR_REQUIRE(ldx >= cols && ldy >= ((flags & TR_LINEAR_EPI_SWIGLU) ? rows / 2 : rows),
             "tr_linear: leading dimensions too small");
  TR_REQUIRE(((uintptr_t)w & 15) == 0, "tr_linear: weight buffer must be 16-byte aligned");
  const int epi = (flags & TR_LINEAR_EPI_SWIGLU) ? 1 : 0;
  const int out_f32 = (flags & TR_LINEAR_OUT_F32) ? 1 : 0;
  TR_REQUIRE(!(epi && out_f32), "tr_linear: TR_LINEAR_OUT_F32 does not combine with the SwiGLU epilogue");
  if (batch == 0) return 0;
  const int pdl = flags & TR_LINEAR_PDL;
  const int uniform = (flags & TR_LINEAR_UNIFORM_SCALE) ? 1 : 0;
  const int knob = (flags >> 8) & 0xFFFF;   // GEMV: CTA count; UMMA: K split (0 = automatic)
  cudaStream_t st = (cudaStream_t)stream;
  const bool aligned = (ldx % 8) == 0 && ((uintptr_t)x & 15) == 0;
  const bool s8 = batch <= 4 && !(flags & TR_LINEAR_GEMV_F16) && gemv_s8_fits((int)batch, (int)rows, (int)cols, fmt) &&
                  (fmt == kFmtTq2 || !prefer_umma(batch, rows, cols) || (flags & TR_LINEAR_FORCE_GEMV));
  if (epi) {   // SwiGLU: the int8-slice GEMV or K5 (the two kernels that know the gate/up tile pairing)
    TR_REQUIRE(fmt == kFmtTq2, "tr_linear: the SwiGLU epilogue takes TQ2 weights");
    const bool umma_epi = aligned && (rows % 32) == 0 && !(flags & (TR_LINEAR_FORCE_GEMV | TR_LINEAR_GEMV_F16)) &&
                          ((flags & TR_LINEAR_FORCE_UMMA) || !s8 || prefer_umma(batch, rows, cols));
    if (umma_epi)
      return gemm_umma(fmt, act_dtype, w, x, y, ldx, ldy, (int)batch, (int)rows, (int)cols, knob, uniform, workspace,
                       ws_bytes, pdl, st, (flags >> 24) & 0xF, 0, 1);
    TR_REQUIRE(s8 && !(flags & TR_LINEAR_FORCE_UMMA),
               "tr_linear: the SwiGLU epilogue runs on the int8-slice GEMV (batch <= 4) or the tensor-core GEMM "
               "(16-byte aligned activation rows, rows a multiple of 32)");
    return gemv_s8(act_dtype, w, x, y, ldx, ldy, (int)batch, (int)rows, (int)cols, knob, pdl, st, 0, nullptr, nullptr,
                   nullptr, 0.0f, sched_mode(flags), 1, 0, kFmtTq2);
  }
  bool use_umma = aligned && (prefer_umma(batch, rows, cols) ||
                               (batch >= 3 && batch <= 8 && !gemv_stages_x((int)batch, (int)rows, (int)cols)));
  if (flags & TR_LINEAR_FORCE_UMMA) {
    TR_REQUIRE(aligned, "tr_linear: the tensor-core path needs 16-byte aligned activation rows");
    use_umma = true;
  }
  if (flags & TR_LINEAR_FORCE_GEMV) use_umma = false;
  if (fmt == kFmtTq1) {   // 1.6-bit weights: K4 (int8 GEMV, batch 1-4) or the tensor-core GEMM
    if (flags & TR_LINEAR_FORCE_GEMV)
      TR_REQUIRE(s8, "tr_linear: the TQ1 GEMV (K4) takes batch 1-4 with activations that fit in shared memory");
    use_umma = !s8 || (flags & TR_LINEAR_FORCE_UMMA);
    TR_REQUIRE(!use_umma || aligned, "tr_linear: TQ1 on the tensor cores needs 16-byte aligned activation rows");
  }
  if (use_umma)
    return gemm_umma(fmt, act_dtype, w, x, y, ldx, ldy, (int)batch, (int)rows, (int)cols, knob, uniform, workspace,
                     ws_bytes, pdl, st, (flags >> 24) & 0xF, out_f32, 0);
  if (s8)
    return gemv_s8(act_dtype, w, x, y, ldx, ldy, (int)batch, (int)rows, (int)cols, knob, pdl, st, 0, nullptr, nullptr,
                   nullptr, 0.0f, sched_mode(flags), 0, out_f32, fmt);
  const size_t esz = 2, ysz = out_f32 ? 4 : 2;
  for (int64_t n0 = 0; n0 < batch; n0 += 32) {
    const int nb_ = (int)(batch - n0 < 32 ? batch - n0 : 32);
    int rc = gemv_tq2(act_dtype, w, (const uint8_t*)x + n0 * ldx * esz, (uint8_t*)y + n0 * ldy * ysz, ldx, ldy, nb_,
                      (int)rows, (int)cols, knob, pdl, st, 0, nullptr, nullptr, nullptr, 0.0f, out_f32);
    if (rc) return rc;
  }
  return 0;
}

int tr_linear_pre(int fmt, const void* w, const void* x, void* y, int64_t batch, int64_t rows, int64_t cols,
                  int act_dtype, int64_t ldx, int64_t ldy, int flags, int pre_op, const void* delta, const void* gamma,
                  void* x_out, float eps, void* stream) {
  TR_REQUIRE(fmt == kFmtTq2, "tr_linear_pre: TQ2 only");
  TR_REQUIRE(act_dtype == kActF16 || act_dtype == kActBf16, "tr_linear_pre: act_dtype must be F16(1) or BF16(2)");
  TR_REQUIRE(pre_op == TR_PRE_ADD_RMSNORM || pre_op == TR_PRE_SILU_MUL, "tr_linear_pre: bad pre_op %d", pre_op);
  TR_REQUIRE(pre_op != TR_PRE_ADD_RMSNORM || gamma != nullptr, "tr_linear_pre: RMSNorm needs gamma");
  TR_REQUIRE(batch >= 1 && batch <= 8 && rows >= 1 && cols >= 1, "tr_linear_pre: 1 <= batch <= 8");
  TR_REQUIRE(ldx >= (pre_op == TR_PRE_SILU_MUL ? 2 * cols : cols) &&
                 ldy >= ((flags & TR_LINEAR_EPI_SWIGLU) ? rows / 2 : rows),
             "tr_linear_pre: leading dimensions");
  TR_REQUIRE(((uintptr_t)w & 15) == 0, "tr_linear_pre: weight buffer must be 16-byte aligned");
  TR_REQUIRE(!(flags & TR_LINEAR_OUT_F32), "tr_linear_pre: TR_LINEAR_OUT_F32 is not supported here");
  if (flags & TR_LINEAR_EPI_SWIGLU)
    TR_REQUIRE(batch <= 4 && !(flags & TR_LINEAR_GEMV_F16) && gemv_s8_fits((int)batch, (int)rows, (int)cols, kFmtTq2),
               "tr_linear_pre: the SwiGLU epilogue runs on the int8-slice GEMV only (batch <= 4)");
  if (batch <= 4 && !(flags & TR_LINEAR_GEMV_F16) && gemv_s8_fits((int)batch, (int)rows, (int)cols, kFmtTq2))
    return gemv_s8(act_dtype, w, x, y, ldx, ldy, (int)batch, (int)rows, (int)cols, (flags >> 8) & 0xFFFF,
                   flags & TR_LINEAR_PDL, (cudaStream_t)stream, pre_op, delta, gamma, x_out, eps,
                   sched_mode(flags), (flags & TR_LINEAR_EPI_SWIGLU) ? 1 : 0, 0, kFmtTq2);
  return gemv_tq2(act_dtype, w, x, y, ldx, ldy, (int)batch, (int)rows, (int)cols, (flags >> 8) & 0xFFFF,
                  flags & TR_LINEAR_PDL, (cudaStream_t)stream, pre_op, delta, gamma, x_out, eps, 0);
}

size_t tr_qkv_attn_decode_workspace_size(int64_t heads) { return heads > 0 ? (size_t)heads * 4 : 0; }

int tr_qkv_attn_decode(int act_dtype, const void* w_qkv, const void* h, const void* delta, const void* gamma,
                       void* h_out, float eps, void* qkv_out, const int64_t* pos, const void* cos_t,
                       const void* sin_t, void* k_cache, void* v_cache, void* att_out, int64_t heads,
                       int64_t head_dim, int64_t max_seq, float scale, void* workspace, size_t ws_bytes, int flags,
                       void* stream) {
  TR_REQUIRE(heads >= 1 && ws_bytes >= tr_qkv_attn_decode_workspace_size(heads),
             "tr_qkv_attn_decode: workspace of %zu bytes, %zu needed", ws_bytes,
             tr_qkv_attn_decode_workspace_size(heads > 0 ? heads : 1));
  TR_REQUIRE(act_dtype == kActF16 || act_dtype == kActBf16, "tr_qkv_attn_decode: act_dtype must be F16(1) or BF16(2)");
  TR_REQUIRE(((uintptr_t)w_qkv & 15) == 0, "tr_qkv_attn_decode: weight buffer must be 16-byte aligned");
  TR_REQUIRE(heads >= 1 && heads * head_dim < (1 << 24), "tr_qkv_attn_decode: bad heads");
  return gemv_qkv_attn(act_dtype, w_qkv, h, delta, gamma, h_out, eps, qkv_out, pos, cos_t, sin_t, k_cache, v_cache,
                       att_out, (int)heads, (int)head_dim, (int)max_seq, scale, workspace, flags & TR_LINEAR_PDL,
                       (flags >> 16) & 0xfff, (cudaStream_t)stream);   // (bits 16..27: dev probes)
}

size_t tr_linear_chain_workspace_size(int64_t n_layers) {
  if (n_layers < 1 || n_layers > 256) return 0;
  return chain_workspace_bytes((int)n_layers);
}

int tr_linear_chain_prepare(const TrChainLayer* layers, int64_t n_layers, int64_t batch, void* workspace,
                            size_t ws_bytes) {
  TR_REQUIRE(layers != nullptr && n_layers >= 1 && n_layers <= 256, "tr_linear_chain_prepare: 1..256 layers");
  return gemv_chain_s8(kActF16, layers, (int)n_layers, (int)batch, workspace, ws_bytes, 0, nullptr, true);
}

int tr_linear_chain(int act_dtype, const TrChainLayer* layers, int64_t n_layers, int64_t batch, int flags,
                    void* workspace, size_t ws_bytes, void* stream) {
  TR_REQUIRE(act_dtype == kActF16 || act_dtype == kActBf16, "tr_linear_chain: act_dtype must be F16(1) or BF16(2)");
  TR_REQUIRE(layers != nullptr && n_layers >= 1 && n_layers <= 256, "tr_linear_chain: 1..256 layers");
  return gemv_chain_s8(act_dtype, layers, (int)n_layers, (int)batch, workspace, ws_bytes, flags, (cudaStream_t)stream,
                       false);
}

}  // extern "C"
