// OpEvo fp32 MatMul family (sm_100a SIMT): the paper's TVM dense schedule
// as a hand-written kernel, so every factor of the
// reference's matmul_space is a real knob:
//
//   N = n1*n2*n3*n4, M = m1*m2*m3*m4, K = k1*k2*k3
//   n1 x m1   CTAs (blockIdx.y, blockIdx.x)
//   n3 x m3   threads per CTA (threadIdx.x = ty * M3 + tx)
//   n2 x m2   virtual-thread tiles per thread, interleaved with stride
//             n3*n4 (m3*m4) so a warp's accesses stay contiguous
//   n4 x m4   per-thread register tile of each virtual-thread tile
//   k1        K chunks staged global -> shared memory
//   k2        register-staging steps per shared chunk
//   k3        K values loaded into registers per step (inner unroll)
//
// C[N][M] = A[N][K] . B[M][K]^T, fp32 in / fp32 accumulate / fp32 out
// (the bf16 family's K-major operand layout).  Tolerance 1e-4 relative.

#ifndef OPEVO_N2
#define OPEVO_N2 1
#endif
#ifndef OPEVO_N3
#define OPEVO_N3 16
#endif
#ifndef OPEVO_N4
#define OPEVO_N4 4
#endif
#ifndef OPEVO_M2
#define OPEVO_M2 1
#endif
#ifndef OPEVO_M3
#define OPEVO_M3 16
#endif
#ifndef OPEVO_M4
#define OPEVO_M4 4
#endif
#ifndef OPEVO_K2
#define OPEVO_K2 4
#endif
#ifndef OPEVO_K3
#define OPEVO_K3 4
#endif

namespace opevo_simt {

constexpr int N2 = OPEVO_N2, N3 = OPEVO_N3, N4 = OPEVO_N4;
constexpr int M2 = OPEVO_M2, M3 = OPEVO_M3, M4 = OPEVO_M4;
constexpr int K2 = OPEVO_K2, K3 = OPEVO_K3;
constexpr int THREADS = N3 * M3;
constexpr int BM = N2 * N3 * N4;          // CTA rows
constexpr int BN = M2 * M3 * M4;          // CTA cols
constexpr int KS = K2 * K3;               // K per shared chunk
constexpr int TM = N2 * N4;               // rows per thread
constexpr int TN = M2 * M4;               // cols per thread
constexpr int PAD = 1;                    // break power-of-two bank strides

static_assert(THREADS >= 1 && THREADS <= 1024, "n3*m3 threads per block must be <= 1024");
static_assert(TM * TN <= 256, "register tile too large");

}  // namespace opevo_simt

extern "C" __global__ void __launch_bounds__(opevo_simt::THREADS)
opevo_sgemm(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
            int rows, int cols, int depth)
{
    using namespace opevo_simt;
    extern __shared__ float smem[];
    // programmatic dependent launch: let the next launch start its prologue,
    // but touch global memory only after the previous grid has completed
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float* As = smem;                         // [KS][BM + PAD], K-major for row broadcasts
    float* Bs = smem + KS * (BM + PAD);       // [KS][BN + PAD]

    const int tid = threadIdx.x;
    const int ty = tid / M3, tx = tid % M3;
    const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BN;
    const size_t boff = (size_t)blockIdx.z;
    A += boff * (size_t)rows * depth;
    B += boff * (size_t)cols * depth;
    C += boff * (size_t)rows * cols;

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

    for (int k0 = 0; k0 < depth; k0 += KS) {              // k1 chunks
        // cooperative staging, coalesced along K
        for (int e = tid; e < BM * KS; e += THREADS) {
            const int r = e / KS, k = e - r * KS;
            As[k * (BM + PAD) + r] = A[(size_t)(row0 + r) * depth + k0 + k];
        }
        for (int e = tid; e < BN * KS; e += THREADS) {
            const int c = e / KS, k = e - c * KS;
            Bs[k * (BN + PAD) + c] = B[(size_t)(col0 + c) * depth + k0 + k];
        }
        __syncthreads();
#pragma unroll 1
        for (int kt = 0; kt < K2; ++kt) {                  // k2 steps
            float a[K3][TM], b[K3][TN];
#pragma unroll
            for (int kk = 0; kk < K3; ++kk) {              // k3 values in registers
                const int k = kt * K3 + kk;
#pragma unroll
                for (int v = 0; v < N2; ++v)
#pragma unroll
                    for (int i = 0; i < N4; ++i)
                        a[kk][v * N4 + i] = As[k * (BM + PAD) + v * (N3 * N4) + ty * N4 + i];
#pragma unroll
                for (int w = 0; w < M2; ++w)
#pragma unroll
                    for (int j = 0; j < M4; ++j)
                        b[kk][w * M4 + j] = Bs[k * (BN + PAD) + w * (M3 * M4) + tx * M4 + j];
            }
#pragma unroll
            for (int kk = 0; kk < K3; ++kk)
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[kk][i], b[kk][j], acc[i][j]);
        }
        __syncthreads();
    }

#pragma unroll
    for (int v = 0; v < N2; ++v)
#pragma unroll
        for (int i = 0; i < N4; ++i) {
            const int r = row0 + v * (N3 * N4) + ty * N4 + i;
#pragma unroll
            for (int w = 0; w < M2; ++w)
#pragma unroll
                for (int j = 0; j < M4; ++j) {
                    const int c = col0 + w * (M3 * M4) + tx * M4 + j;
                    C[(size_t)r * cols + c] = acc[v * N4 + i][w * M4 + j];
                }
        }
}
