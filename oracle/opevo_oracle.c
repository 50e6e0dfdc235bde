/*
 * CPU oracle for the B200 evaluator -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  The product path
 * (libopevo.so) never calls it.
 *
 * It restates:
 *  - the synthetic operand generator of libopevo (util_kernels.cu): bit-exact
 *    U(-1,1) values from splitmix64(seed * GOLDEN + i) >> 40, rounded to bf16
 *    with round-to-nearest-even;
 *  - the operators of the paper in fp64:
 *      MatMul  Z[n,m] = sum_k X[n,k] Y[k,m]
 *      BMM     Z[b,n,m] = sum_k X[b,n,k] Y[b,k,m]
 *      Conv2d  direct convolution, NCHW x OIHW
 *    with Y stored K-major ([m][k]) exactly as the kernels consume it.
 *
 * Parity status: the reference package has no operator numerics
 * (benchmarks.py:12-17), so these are pinned to the paper's
 * definitions and to numpy/torch fp64 on the same inputs (tests), not to
 * reference outputs.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static float hashed_uniform(uint64_t seed, uint64_t i) {
    uint64_t h = mix64(seed * 0x9E3779B97F4A7C15ull + i);
    return (float)(h >> 40) * (1.0f / 8388608.0f) - 1.0f;
}

static uint16_t bf16_rne(float f) {
    union { float f; uint32_t u; } v = {f};
    uint32_t b = v.u;
    b += 0x7FFFu + ((b >> 16) & 1u);
    return (uint16_t)(b >> 16);
}

static float bf16_val(uint16_t h) {
    union { uint32_t u; float f; } v = {((uint32_t)h) << 16};
    return v.f;
}

/* operands as the kernels see them: bf16 bits (as float values) or fp32 */
void oracle_fill(float* out, uint64_t n, uint64_t seed, int as_bf16) {
    for (uint64_t i = 0; i < n; ++i) {
        float x = hashed_uniform(seed, i);
        out[i] = as_bf16 ? bf16_val(bf16_rne(x)) : x;
    }
}

void oracle_fill_bf16_bits(uint16_t* out, uint64_t n, uint64_t seed) {
    for (uint64_t i = 0; i < n; ++i) out[i] = bf16_rne(hashed_uniform(seed, i));
}

/* R[b][r][c] = sum_k A[b][r][k] * B[b][c][k] in fp64 */
static void gemm_row(const float* A, const float* B, double* out, int64_t rows, int64_t cols,
                     int64_t depth, int64_t br) {
    const int64_t b = br / rows;
    const float* a = A + br * depth;
    for (int64_t c = 0; c < cols; ++c) {
        const float* y = B + (b * cols + c) * depth;
        double acc = 0.0;
        for (int64_t k = 0; k < depth; ++k) acc += (double)a[k] * (double)y[k];
        out[c] = acc;
    }
}

/* R[b][r][c] = sum_k A[b][r][k] * B[b][c][k] in fp64 (rows in parallel) */
void oracle_gemm(const float* A, const float* B, double* R, int64_t batch, int64_t rows,
                 int64_t cols, int64_t depth) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t br = 0; br < batch * rows; ++br) gemm_row(A, B, R + br * cols, rows, cols, depth, br);
}

/* The same for a sample of output rows: out[i][c] = R[row_idx[i]][c], where
 * row_idx counts rows over all batches (b * rows + r). */
void oracle_gemm_rows(const float* A, const float* B, double* out, int64_t rows, int64_t cols,
                      int64_t depth, const int64_t* row_idx, int64_t nidx) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < nidx; ++i) gemm_row(A, B, out + i * cols, rows, cols, depth, row_idx[i]);
}

/* direct conv, X NCHW, W OIHW -> R NHWC (the implicit-GEMM output layout) */
void oracle_conv(const float* X, const float* W, double* R, int N, int C, int H, int Wd, int K,
                 int KH, int KW, int stride, int pad) {
    const int HO = (H + 2 * pad - KH) / stride + 1, WO = (Wd + 2 * pad - KW) / stride + 1;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int n = 0; n < N; ++n)
        for (int ho = 0; ho < HO; ++ho)
            for (int wo = 0; wo < WO; ++wo)
                for (int k = 0; k < K; ++k) {
                    double acc = 0.0;
                    for (int c = 0; c < C; ++c)
                        for (int i = 0; i < KH; ++i) {
                            const int h = ho * stride - pad + i;
                            if (h < 0 || h >= H) continue;
                            for (int j = 0; j < KW; ++j) {
                                const int w = wo * stride - pad + j;
                                if (w < 0 || w >= Wd) continue;
                                acc += (double)X[(((int64_t)n * C + c) * H + h) * Wd + w] *
                                       (double)W[(((int64_t)k * C + c) * KH + i) * KW + j];
                            }
                        }
                    R[(((int64_t)n * HO + ho) * WO + wo) * K + k] = acc;
                }
}

/* max |C - R| and max |R| over n elements (C widened to double) */
void oracle_compare(const float* Cv, const double* R, uint64_t n, double* max_diff, double* max_ref,
                    uint64_t* nonfinite) {
    double md = 0.0, mr = 0.0;
    uint64_t bad = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (!isfinite(Cv[i])) { ++bad; continue; }
        double d = fabs((double)Cv[i] - R[i]);
        if (d > md) md = d;
        if (fabs(R[i]) > mr) mr = fabs(R[i]);
    }
    *max_diff = md;
    *max_ref = mr;
    *nonfinite = bad;
}
