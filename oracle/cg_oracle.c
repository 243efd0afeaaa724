/*
 * cg_oracle.c -- C restatement of the reference CodeGEMM CPU path.
 * TEST INFRASTRUCTURE ONLY: loaded by tests/ (fast full-size parity) and by
 * bench.py's CPU-baseline leg.  The product library never links it.
 *
 * Restates /root/reference/pkg/src/codegemm/engines.py:
 *   cgo_psum_tables  <- _psum_tables           (engines.py:115-134)
 *   cgo_codegemm     <- codegemm_gemm/consume  (engines.py:245-316, 286-294)
 * with the reference's canonical binary32 operation order (engines.py:15-22):
 *   psum    = ((+0 + c0*x0) + c1*x1) + ...         k ascending
 *   seg_sum = ((+0 + P_0) + P_1) + ...             codebook t ascending
 *   y      += scale * seg_sum                      segments ascending
 * Compiled with -ffp-contract=off so mul and add round separately.  The
 * products c*x of two binary16 values are exact in binary32, so the psum
 * chain equals the reference bit for bit.
 *
 * Output bits do not depend on t_w, t_h or threads (engines.py:15-22), so the
 * threaded version partitions rows across pthreads.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* exact binary16 -> binary32 widening (tensors.py:132-134 "widened") */
static float h2f(uint16_t h) {
    uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    uint32_t exp = (h >> 10) & 0x1fu;
    uint32_t man = h & 0x3ffu;
    uint32_t bits;
    if (exp == 0) {
        if (man == 0) {
            bits = sign;
        } else { /* subnormal: normalise */
            int e = -1;
            do { man <<= 1; ++e; } while ((man & 0x400u) == 0);
            man &= 0x3ffu;
            bits = sign | ((uint32_t)(127 - 15 - e) << 23) | (man << 13);
        }
    } else if (exp == 31) {
        bits = sign | 0x7f800000u | (man << 13);
    } else {
        bits = sign | ((exp + 112u) << 23) | (man << 13);
    }
    float f;
    memcpy(&f, &bits, sizeof f);
    return f;
}

void cgo_widen_f16(const uint16_t* in, float* out, int64_t count) {
    for (int64_t i = 0; i < count; ++i) out[i] = h2f(in[i]);
}

/* tables[t][j][i][c], j over `segs` segments starting at element `start` */
static void build_tables(const float* const* books32, const float* x32, int m, int kcount,
                         int v, int64_t start, int64_t segs, int n, float* tables) {
    for (int t = 0; t < m; ++t) {
        const float* c = books32[t];
        for (int64_t j = 0; j < segs; ++j) {
            float* tab = tables + (((int64_t)t * segs + j) * kcount) * n;
            for (int i = 0; i < kcount; ++i) {
                for (int col = 0; col < n; ++col) {
                    float acc = 0.0f;
                    for (int kk = 0; kk < v; ++kk) {
                        float prod = c[(int64_t)i * v + kk] * x32[(start + j * v + kk) * n + col];
                        acc = acc + prod;
                    }
                    tab[(int64_t)i * n + col] = acc;
                }
            }
        }
    }
}

/* (m, K/v, 2**b, n) float32; x is (K, n) binary16 bits, books m x (2**b, v) */
int cgo_psum_tables(const uint16_t* const* books, const uint16_t* x, int m, int b, int v,
                    int64_t k_len, int n, float* out) {
    if (m < 1 || b < 1 || b > 16 || v < 1 || k_len % v || n < 1) return 1;
    int kcount = 1 << b;
    float** books32 = (float**)calloc((size_t)m, sizeof(float*));
    float* x32 = (float*)malloc(sizeof(float) * (size_t)(k_len * n));
    cgo_widen_f16(x, x32, k_len * n);
    for (int t = 0; t < m; ++t) {
        books32[t] = (float*)malloc(sizeof(float) * (size_t)kcount * v);
        cgo_widen_f16(books[t], books32[t], (int64_t)kcount * v);
    }
    build_tables((const float* const*)books32, x32, m, kcount, v, 0, k_len / v, n, out);
    for (int t = 0; t < m; ++t) free(books32[t]);
    free(books32);
    free(x32);
    return 0;
}

typedef struct {
    const uint16_t* const* codes;
    const float* const* books32;
    const float* x32;
    const float* scales32;
    int m, kcount, n, v, t_w;
    int64_t cols, segs_total, groups, g_eff;
    int64_t r0, r1;
    float* y;
} rows_args;

/*
 * One worker: every K-tile in ascending order (engines.py:298), build the
 * tile tables (engines.py:299, private copy per worker -- bits are identical),
 * then consume its rows (engines.py:286-294).
 */
static void* run_rows(void* p) {
    rows_args* a = (rows_args*)p;
    int n = a->n, m = a->m, kcount = a->kcount, v = a->v;
    int64_t max_tile_segs = a->t_w / v;
    float* tables = (float*)malloc(sizeof(float) * (size_t)m * max_tile_segs * kcount * n);
    float* seg_sum = (float*)malloc(sizeof(float) * (size_t)n);
    for (int64_t start = 0; start < a->cols; start += a->t_w) {
        int64_t width = (a->cols - start < a->t_w) ? a->cols - start : a->t_w;
        int64_t tile_segs = width / v, seg0 = start / v;
        build_tables(a->books32, a->x32, m, kcount, v, start, tile_segs, n, tables);
        for (int64_t r = a->r0; r < a->r1; ++r) {
            float* yr = a->y + r * n;
            for (int64_t j = 0; j < tile_segs; ++j) {
                int64_t seg = seg0 + j;
                for (int c = 0; c < n; ++c) seg_sum[c] = 0.0f;
                for (int t = 0; t < m; ++t) {
                    uint16_t code = a->codes[t][r * a->segs_total + seg];
                    const float* ent = tables + (((int64_t)t * tile_segs + j) * kcount + code) * n;
                    for (int c = 0; c < n; ++c) seg_sum[c] = seg_sum[c] + ent[c];
                }
                float s = a->scales32[r * a->groups + (seg * v) / a->g_eff];
                for (int c = 0; c < n; ++c) {
                    float prod = s * seg_sum[c];
                    yr[c] = yr[c] + prod;
                }
            }
        }
    }
    free(seg_sum);
    free(tables);
    return NULL;
}

/*
 * y (rows, n) float32 = codegemm_gemm(q, x, TileConfig(t_w, *), threads)[0].
 * codes: m planes (rows, K/v) uint16; books: m (2**b, v) f16 bits;
 * scales: (rows, K/g_eff) f16 bits; x: (K, n) f16 bits; g = -1 for per-row.
 */
int cgo_codegemm(const uint16_t* const* codes, const uint16_t* const* books,
                 const uint16_t* scales, const uint16_t* x, int64_t rows, int64_t cols,
                 int v, int m, int b, int64_t g, int n, int t_w, int threads, float* y) {
    if (rows < 1 || cols < 1 || v < 1 || m < 1 || b < 1 || b > 16 || n < 1) return 1;
    if (cols % v || t_w < v || t_w % v) return 1;
    int64_t g_eff = (g == -1) ? cols : g;
    if (g_eff < 1 || cols % g_eff) return 1;
    if (threads < 1) threads = 1;
    int kcount = 1 << b;
    int64_t segs = cols / v, groups = cols / g_eff;

    float* x32 = (float*)malloc(sizeof(float) * (size_t)(cols * n));
    float* scales32 = (float*)malloc(sizeof(float) * (size_t)(rows * groups));
    float** books32 = (float**)calloc((size_t)m, sizeof(float*));
    cgo_widen_f16(x, x32, cols * n);
    cgo_widen_f16(scales, scales32, rows * groups);
    for (int t = 0; t < m; ++t) {
        books32[t] = (float*)malloc(sizeof(float) * (size_t)kcount * v);
        cgo_widen_f16(books[t], books32[t], (int64_t)kcount * v);
    }
    memset(y, 0, sizeof(float) * (size_t)(rows * n));

    pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    rows_args* args = (rows_args*)malloc(sizeof(rows_args) * (size_t)threads);
    int64_t per = (rows + threads - 1) / threads;
    int used = 0;
    for (int th = 0; th < threads; ++th) {
        int64_t r0 = th * per, r1 = r0 + per < rows ? r0 + per : rows;
        if (r0 >= r1) break;
        rows_args a = {codes, (const float* const*)books32, x32, scales32, m, kcount, n, v, t_w,
                       cols, segs, groups, g_eff, r0, r1, y};
        args[th] = a;
        ++used;
    }
    if (used == 1) {
        run_rows(&args[0]);
    } else {
        for (int th = 0; th < used; ++th) pthread_create(&tids[th], NULL, run_rows, &args[th]);
        for (int th = 0; th < used; ++th) pthread_join(tids[th], NULL);
    }
    free(args);
    free(tids);
    for (int t = 0; t < m; ++t) free(books32[t]);
    free(books32);
    free(scales32);
    free(x32);
    return 0;
}
