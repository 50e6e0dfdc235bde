// Does a tcgen05 SW128 K-major operand descriptor accept a start address that
// is a whole number of 128-byte rows past a 1024-byte swizzle atom, and with
// which "matrix base offset" (descriptor bits 49-51)?  (Decides whether a conv
// halo box can serve three filter taps by shifting the A descriptor one row
// per tap.)  A is written by threads in the TMA SW128 pattern keyed on the
// absolute shared address; D = A[s..s+127] . B^T is read back from TMEM and
// compared with the host product for s = 0..9 and base offset 0 or s & 7;
// then with 8-row groups L rows apart (SBO = L * 128 B, L = 8, 10, 12, 16),
// i.e. MMA row r = smem row (r / 8) * L + r % 8 + s -- a halo box whose lines
// are TILE_W + 2 pixels wide.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/swizzle_probe tools/swizzle_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

typedef unsigned int u32;
typedef unsigned long long u64;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

// A: AROWS rows x 64 bf16 (one 128-byte swizzle row each), B: 64 rows x 64 bf16
#define AROWS 288
__global__ void __launch_bounds__(128, 1) probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D,
                                                int shift, int base_mode, int lrows) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    __shared__ __align__(8) u64 bar;
    __shared__ u32 tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u32 a0 = smem_u32(smem), b0 = a0 + AROWS * 128;
    // stage A and B in the SW128 pattern: 16-byte chunk j of row r lands at
    // chunk j ^ (r & 7), r counted from the 1024-aligned base
    for (int c = threadIdx.x; c < AROWS * 8; c += blockDim.x) {
        const int r = c >> 3, j = c & 7;
        const uint4 v = *reinterpret_cast<const uint4*>(A + r * 64 + j * 8);
        *reinterpret_cast<uint4*>(smem + r * 128 + ((j ^ (r & 7)) << 4)) = v;
    }
    for (int c = threadIdx.x; c < 64 * 8; c += blockDim.x) {
        const int r = c >> 3, j = c & 7;
        const uint4 v = *reinterpret_cast<const uint4*>(B + r * 64 + j * 8);
        *reinterpret_cast<uint4*>(smem + AROWS * 128 + r * 128 + ((j ^ (r & 7)) << 4)) = v;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" :: "r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = tslot;
    constexpr u32 IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((u32)(64 >> 3) << 17) | ((u32)(128 >> 4) << 24);
    const u64 HI = ((u64)1 << 16) | ((u64)((lrows * 128) >> 4) << 32) | ((u64)1 << 46) | ((u64)2 << 61);
    const u64 base_off = base_mode ? (u64)(shift & 7) : 0;
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const u64 ad = HI | (base_off << 49) | (u64)(((a0 + shift * 128 + k * 32) >> 4) & 0x3FFF);
            const u64 bd = HI | (u64)(((b0 + k * 32) >> 4) & 0x3FFF);
            const u32 acc = k ? 1u : 0u;
            asm volatile("{ .reg .pred e, p; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; "
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                         :: "r"(tmem), "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
        }
        asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }"
                     :: "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }"
                 :: "r"(smem_u32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    u32 v[32];
    for (int half = 0; half < 2; ++half) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                       "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                       "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(tmem + ((u32)(warp * 32) << 16) + (u32)(half * 32)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int row = warp * 32 + lane;
        for (int c = 0; c < 32; ++c) D[row * 64 + half * 32 + c] = __uint_as_float(v[c]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tmem));
}

int main() {
    const int AR = AROWS, BR = 64, K = 64;
    __nv_bfloat16 *hA = new __nv_bfloat16[AR * K], *hB = new __nv_bfloat16[BR * K];
    float* fa = new float[AR * K];
    float* fb = new float[BR * K];
    for (int r = 0; r < AR; ++r)
        for (int k = 0; k < K; ++k) { fa[r * K + k] = (float)((r * 7 + k * 3) % 9 - 4); hA[r * K + k] = __float2bfloat16(fa[r * K + k]); }
    for (int r = 0; r < BR; ++r)
        for (int k = 0; k < K; ++k) { fb[r * K + k] = (float)((r * 5 + k * 11) % 7 - 3); hB[r * K + k] = __float2bfloat16(fb[r * K + k]); }
    __nv_bfloat16 *dA, *dB;
    float* dD;
    cudaMalloc(&dA, AR * K * 2);
    cudaMalloc(&dB, BR * K * 2);
    cudaMalloc(&dD, 128 * 64 * 4);
    cudaMemcpy(dA, hA, AR * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, BR * K * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    float* hD = new float[128 * 64];
    struct Case { int mode, lrows, smax; };
    const Case cases[] = {{0, 8, 9}, {1, 8, 9}, {0, 10, 2}, {0, 12, 2}, {0, 16, 2}};
    for (const Case& cs : cases) {
        for (int s = 0; s <= cs.smax; ++s) {
            cudaMemset(dD, 0, 128 * 64 * 4);
            probe<<<1, 128, 80 * 1024>>>(dA, dB, dD, s, cs.mode, cs.lrows);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("shift %d base_mode %d: CUDA error %s\n", s, cs.mode, cudaGetErrorString(e)); return 1; }
            cudaMemcpy(hD, dD, 128 * 64 * 4, cudaMemcpyDeviceToHost);
            int bad = 0, bad_r0 = -1;
            for (int r = 0; r < 128; ++r)
                for (int n = 0; n < 64; ++n) {
                    const int ar = (r / 8) * cs.lrows + r % 8 + s;
                    float ref = 0.f;
                    for (int k = 0; k < K; ++k) ref += fa[ar * K + k] * fb[n * K + k];
                    if (hD[r * 64 + n] != ref) { if (bad_r0 < 0) bad_r0 = r; ++bad; }
                }
            printf("SBO %2d rows, shift %d rows, base offset %s: %s (%d wrong, first wrong row %d)\n", cs.lrows, s,
                   cs.mode ? "= shift & 7" : "= 0       ", bad ? "MISMATCH" : "exact", bad, bad_r0);
        }
    }
    return 0;
}
