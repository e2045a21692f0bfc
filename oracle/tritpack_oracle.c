/*
 * oracle/tritpack_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU kernels of the TriRun hot path
 * (the `tritpack` package, /root/reference/pkg/src/tritpack/_kernels.pyx and
 * its numpy twin _kernels_py.py).  It is the *checker*: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product (paper_2506_23025_b200) never links or calls it.
 *
 * Parity of this restatement is pinned against the reference itself:
 *   - the tests/golden fixtures were produced by importing the reference package
 *     (tests/golden/make_golden.py) and are checked bit-for-bit by
 *     tests/test_oracle.py;
 *   - oracle/_ref/ holds the reference's own compiled kernels (Cython -> C,
 *     built by oracle/Makefile straight from the reference sources) and
 *     tests/test_oracle.py compares the two on random inputs.
 *
 * Arithmetic contract (reference _kernels_py.py:1-30): digits d = trit + 1 in
 * {0,1,2}; quantize with float32 absmax and float32 reciprocal; dequantize
 * scale * (d - 1); matmul builds +x / -x / +0.0 terms, collapses each
 * 256-term block with a fixed adjacent-pair tree, then acc = acc + s * T in
 * float32, blocks ascending, no FMA (compile with -ffp-contract=off).
 */
#include <stdint.h>
#include <stddef.h>

#define BLK 256
#define TQ2_PB 64
#define TQ1_PB 52

/* reference: _kernels.pyx:23-35 (pack_base4), element 4t+j at bits 2j */
void orc_pack_base4(const uint8_t *digits, uint8_t *out, int64_t m) {
    for (int64_t i = 0; i < m; ++i) {
        const uint8_t *d = digits + 4 * i;
        out[i] = (uint8_t)(d[0] | (d[1] << 2) | (d[2] << 4) | (d[3] << 6));
    }
}

/* reference: _kernels.pyx:38-52 (unpack_base4) */
void orc_unpack_base4(const uint8_t *words, uint8_t *out, int64_t m) {
    for (int64_t i = 0; i < m; ++i)
        for (int j = 0; j < 4; ++j) out[4 * i + j] = (words[i] >> (2 * j)) & 3;
}

/* reference: _kernels.pyx:55-70 (encode_base3): N read MSB-first,
 * code = (N*256 + 242) // 243 */
void orc_encode_base3(const uint8_t *digits, uint8_t *out, int64_t m) {
    for (int64_t i = 0; i < m; ++i) {
        uint32_t n = 0;
        for (int j = 0; j < 5; ++j) n = n * 3u + digits[5 * i + j];
        out[i] = (uint8_t)((n * 256u + 242u) / 243u);
    }
}

/* reference: _kernels.pyx:73-87 (decode_base3) = paper Algorithm 1
 * (PAPER.md:919-937): 5x {p = s*3; d = p >> 8; s = p & 0xFF}. */
void orc_decode_base3(const uint8_t *codes, uint8_t *out, int64_t m) {
    for (int64_t i = 0; i < m; ++i) {
        uint32_t s = codes[i];
        for (int j = 0; j < 5; ++j) {
            uint32_t p = s * 3u;
            out[5 * i + j] = (uint8_t)(p >> 8);
            s = p & 0xFFu;
        }
    }
}

/* reference: _kernels.pyx:90-118 (quantize_blocks), rules _kernels_py.py:10-15 */
void orc_quantize_blocks(const float *values, uint8_t *digits, float *scales, int64_t nb) {
    for (int64_t b = 0; b < nb; ++b) {
        const float *v = values + b * BLK;
        float am = 0.0f;
        for (int t = 0; t < BLK; ++t) {
            float a = v[t] < 0.0f ? -v[t] : v[t];
            if (a > am) am = a;
        }
        float inv = am > 0.0f ? 1.0f / am : 0.0f;
        scales[b] = am;
        for (int t = 0; t < BLK; ++t) {
            float q = v[t] * inv;
            digits[b * BLK + t] = (uint8_t)(q >= 0.5f ? 2 : (q <= -0.5f ? 0 : 1));
        }
    }
}

/* reference: _kernels.pyx:121-133 (dequantize_blocks): (float(d) - 1) * scale */
void orc_dequantize_blocks(const uint8_t *digits, const float *scales, float *out, int64_t nb) {
    for (int64_t b = 0; b < nb; ++b)
        for (int t = 0; t < BLK; ++t)
            out[b * BLK + t] = ((float)digits[b * BLK + t] - 1.0f) * scales[b];
}

/* reference: _kernels.pyx:136-168 (_accumulate_row).  dg: digits of one
 * packed row (nb x 256); the 256-leaf tree is t[i] <- t[2i] + t[2i+1]. */
static void accumulate_row(const uint8_t *dg, const float *srow, const float *x,
                           float *out, int64_t rows, int64_t r, int64_t nb,
                           int64_t batch) {
    float terms[BLK];
    for (int64_t j = 0; j < batch; ++j) {
        const float *xj = x + j * nb * BLK;
        float acc = 0.0f;
        for (int64_t b = 0; b < nb; ++b) {
            for (int t = 0; t < BLK; ++t) {
                uint8_t d = dg[b * BLK + t];
                float xv = xj[b * BLK + t];
                terms[t] = d == 2 ? xv : (d == 0 ? -xv : 0.0f);
            }
            for (int w = BLK / 2; w >= 1; w >>= 1)
                for (int t = 0; t < w; ++t) terms[t] = terms[2 * t] + terms[2 * t + 1];
            float prod = srow[b] * terms[0];
            acc = acc + prod;
        }
        out[j * rows + r] = acc;
    }
}

/* reference: _kernels.pyx:171-197 (gemm_tq2).  payload (rows, nb, 64),
 * scales f32 (rows, nb), x f32 (batch, nb*256), out f32 (batch, rows);
 * rows [row0, row1) are written.  dg_scratch holds nb*256 bytes. */
void orc_gemm_tq2(const uint8_t *payload, const float *scales, const float *x,
                  float *out, int64_t rows, int64_t nb, int64_t batch,
                  int64_t row0, int64_t row1, uint8_t *dg_scratch) {
    for (int64_t r = row0; r < row1; ++r) {
        const uint8_t *p = payload + r * nb * TQ2_PB;
        for (int64_t i = 0; i < nb * TQ2_PB; ++i)
            for (int j = 0; j < 4; ++j) dg_scratch[4 * i + j] = (p[i] >> (2 * j)) & 3;
        accumulate_row(dg_scratch, scales + r * nb, x, out, rows, r, nb, batch);
    }
}

/* reference: _kernels.pyx:200-227 (gemm_tq1): per block 52 codes decode
 * to 260 digits of which the first 256 are real. */
void orc_gemm_tq1(const uint8_t *payload, const float *scales, const float *x,
                  float *out, int64_t rows, int64_t nb, int64_t batch,
                  int64_t row0, int64_t row1, uint8_t *dg_scratch) {
    for (int64_t r = row0; r < row1; ++r) {
        for (int64_t b = 0; b < nb; ++b) {
            const uint8_t *p = payload + (r * nb + b) * TQ1_PB;
            uint8_t *dst = dg_scratch + b * BLK;
            for (int c = 0; c < TQ1_PB; ++c) {
                uint32_t s = p[c];
                for (int j = 0; j < 5; ++j) {
                    uint32_t prod = s * 3u;
                    int idx = 5 * c + j;
                    if (idx < BLK) dst[idx] = (uint8_t)(prod >> 8);
                    s = prod & 0xFFu;
                }
            }
        }
        accumulate_row(dg_scratch, scales + r * nb, x, out, rows, r, nb, batch);
    }
}

/* reference: linear.py:177-208 (dequantize_matrix + gemv_reference) for large
 * shapes: out[j, r] = sum_k f64(scale[r, k / 256]) * (digit(r, k) - 1) * x[j, k]
 * in float64, without materialising the dense matrix.  Digits as dequantize_matrix
 * decodes them: TQ2 by shifts (:184-186), TQ1 by the canonical division formula
 * x = (c * 243 + 13) >> 8, d_j = (x // 3^(4-j)) % 3 (:189-192).  Scales are binary16
 * bit patterns (PackedMatrix.scales).  Rows [row0, row1), x: [batch, cols] float64. */
static double f16_to_f64(uint16_t h) {
    const int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0) v = m * (1.0 / 16777216.0);               /* m * 2^-24 */
    else if (e == 31) v = m ? (0.0 / 0.0) : (1.0 / 0.0);
    else {
        v = 1.0 + m / 1024.0;
        for (int i = 15; i < e; ++i) v *= 2.0;
        for (int i = e; i < 15; ++i) v *= 0.5;
    }
    return s ? -v : v;
}

void orc_gemv_f64(int fmt, const uint8_t *payload, const uint16_t *scales, const double *x, double *out,
                  int64_t rows, int64_t cols, int64_t batch, int64_t row0, int64_t row1) {
    const int64_t nb = (cols + BLK - 1) / BLK;
    const int pb = fmt == 2 ? TQ2_PB : TQ1_PB;
    static const uint32_t pw[5] = {81, 27, 9, 3, 1};
    for (int64_t r = row0; r < row1; ++r) {
        for (int64_t j = 0; j < batch; ++j) out[j * rows + r] = 0.0;
        for (int64_t b = 0; b < nb; ++b) {
            const uint8_t *p = payload + (r * nb + b) * pb;
            const double s = f16_to_f64(scales[r * nb + b]);
            int8_t t[260];
            if (fmt == 2) {
                for (int i = 0; i < TQ2_PB; ++i)
                    for (int q = 0; q < 4; ++q) t[4 * i + q] = (int8_t)((p[i] >> (2 * q)) & 3) - 1;
            } else {
                for (int i = 0; i < TQ1_PB; ++i) {
                    const uint32_t xq = ((uint32_t)p[i] * 243u + 13u) >> 8;
                    for (int q = 0; q < 5; ++q) t[5 * i + q] = (int8_t)((xq / pw[q]) % 3) - 1;
                }
            }
            const int64_t k0 = b * BLK, kn = (cols - k0) < BLK ? (cols - k0) : BLK;
            for (int64_t j = 0; j < batch; ++j) {
                const double *xr = x + j * cols + k0;
                double acc = 0.0;
                for (int64_t k = 0; k < kn; ++k) acc += (s * t[k]) * xr[k];
                out[j * rows + r] += acc;
            }
        }
    }
}
