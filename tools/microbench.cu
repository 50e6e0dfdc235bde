// Microbenchmarks that size the 1024^3 GEMM design (not product code).
//   mma  : cycles per tcgen05.mma.kind::f16 (SS operands, M=128) for N in {64,128,256},
//          issued back to back by one thread, no barriers in the loop.
//   bulk : per-SM and chip-wide cp.async.bulk (TMA) ingress from an L2-resident
//          buffer, as a function of the number of CTAs and the bytes in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/microbench tools/microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

typedef unsigned int u32;
typedef unsigned long long u64;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ u64 gtimer() { u64 t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                 :: "r"(bar), "r"(parity) : "memory");
}

template <int N>
__global__ void __launch_bounds__(128, 1) mma_bench(u64* out, int iters) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    __shared__ u64 bar;
    __shared__ u32 tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (128 + 256) * 64 * 2 / 4; i += blockDim.x) ((u32*)smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = tslot;
    constexpr u32 IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((u32)(N >> 3) << 17) | ((u32)(128 >> 4) << 24);
    constexpr u64 HI = ((u64)1 << 16) | ((u64)(1024 >> 4) << 32) | ((u64)1 << 46) | ((u64)2 << 61);
    const u32 a0 = smem_u32(smem), b0 = a0 + 128 * 128;
    if (warp == 0) {
        u64 t0 = 0, t1 = 0, c0 = 0, c1 = 0;
        for (int rep = 0; rep < 2; ++rep) {       // rep 0 warms up
            c0 = clock64(); t0 = gtimer();
            for (int i = 0; i < iters; ++i) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const u64 ad = HI | (u64)(((a0 + k * 32) >> 4) & 0x3FFF);
                    const u64 bd = HI | (u64)(((b0 + k * 32) >> 4) & 0x3FFF);
                    const u32 acc = (i | k) ? 1u : 0u;
                    asm volatile("{ .reg .pred e, p; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; "
                                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                                 :: "r"(tmem), "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
                }
            }
            asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }"
                         :: "r"(smem_u32(&bar)) : "memory");
            mbar_wait(smem_u32(&bar), rep & 1);
            c1 = clock64(); t1 = gtimer();
        }
        if (threadIdx.x == 0) {
            out[blockIdx.x * 2] = c1 - c0;
            out[blockIdx.x * 2 + 1] = t1 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tmem));
}

// Each CTA streams `per_cta` bytes from src (offset by its index modulo
// `wrap`) into a ring of `stages` x `chunk` bytes of shared memory.
__global__ void __launch_bounds__(32, 1) bulk_bench(const char* src, size_t per_cta, size_t wrap, int chunk,
                                                    int stages, u64* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ u64 bars[16];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&bars[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const char* base = src + ((size_t)blockIdx.x * per_cta) % wrap;
    const int n = (int)(per_cta / chunk);
    u64 c0 = clock64(), t0 = gtimer();
    if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) {
            const int s = i % stages;
            if (i >= stages) mbar_wait(smem_u32(&bars[s]), ((i / stages) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bars[s])), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(smem_u32(smem + s * chunk)), "l"(base + (size_t)i * chunk), "r"(chunk),
                            "r"(smem_u32(&bars[s])) : "memory");
        }
        for (int i = n; i < n + stages && i >= stages; ++i) {
            const int s = i % stages;
            mbar_wait(smem_u32(&bars[s]), ((i / stages) - 1) & 1);
        }
    }
    __syncwarp();
    u64 c1 = clock64(), t1 = gtimer();
    if (threadIdx.x == 0) {
        out[blockIdx.x * 2] = c1 - c0;
        out[blockIdx.x * 2 + 1] = t1 - t0;
    }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int N>
void run_mma(u64* d_out, int grid) {
    const int smem = (128 + 256) * 64 * 2 + 1024;
    CK(cudaFuncSetAttribute(mma_bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int iters = 256;
    mma_bench<N><<<grid, 128, smem>>>(d_out, iters);
    CK(cudaDeviceSynchronize());
    u64 h[2 * 148];
    CK(cudaMemcpy(h, d_out, sizeof(u64) * 2 * grid, cudaMemcpyDeviceToHost));
    double cyc = 0, ns = 0;
    for (int i = 0; i < grid; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; }
    cyc /= grid; ns /= grid;
    const int mmas = iters * 4;
    const double flop = 2.0 * 128 * N * 16 * mmas;
    printf("mma M=128 N=%3d grid=%3d: %.1f cyc/MMA (ideal %d), %.2f GHz, %.2f TFLOP/s/SM -> %.0f TFLOP/s x148\n",
           N, grid, cyc / mmas, 128 * N / 256, cyc / ns, flop / ns / 1e3, 148 * flop / ns / 1e3);
}

int main() {
    u64* d_out;
    CK(cudaMalloc(&d_out, sizeof(u64) * 2 * 1024));
    for (int g : {1, 148}) {
        run_mma<64>(d_out, g);
        run_mma<128>(d_out, g);
        run_mma<256>(d_out, g);
    }
    const size_t buf = 32ull << 20;   // L2-resident source
    char* src;
    CK(cudaMalloc(&src, buf));
    CK(cudaMemset(src, 1, buf));
    CK(cudaFuncSetAttribute(bulk_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    const size_t per_cta = 384 * 1024;
    for (int inflight_kb : {32, 64, 128, 192}) {
        for (int chunk : {8192, 16384}) {
            const int stages = inflight_kb * 1024 / chunk;
            if (stages < 2 || stages > 16) continue;
            for (int grid : {1, 16, 64, 128, 148}) {
                for (int rep = 0; rep < 2; ++rep)
                    bulk_bench<<<grid, 32, stages * chunk + 1024>>>(src, per_cta, buf, chunk, stages, d_out);
                CK(cudaDeviceSynchronize());
                u64 h[2 * 148];
                CK(cudaMemcpy(h, d_out, sizeof(u64) * 2 * grid, cudaMemcpyDeviceToHost));
                double cyc = 0, ns = 0, mx = 0;
                for (int i = 0; i < grid; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; if (h[2 * i + 1] > mx) mx = h[2 * i + 1]; }
                cyc /= grid; ns /= grid;
                printf("bulk inflight=%3d KB chunk=%5d grid=%3d: %.1f B/clk/SM, %.1f GB/s/SM, chip %.2f TB/s (slowest CTA %.2f us)\n",
                       inflight_kb, chunk, grid, per_cta / cyc, per_cta / ns, grid * per_cta / mx / 1e3, mx / 1e3);
            }
        }
    }
    return 0;
}
