// Tensor-TMA ingress microbenchmark (not product code): the GEMM mainloop's
// load pattern without the MMA.  Each CTA streams an A tile (a_rows x K) and
// a B tile (b_rows x K) of L2-resident bf16 matrices through a ring of
// `stages` stages of BK columns (128-byte swizzled boxes of 64 x rows), the
// way opevo_gemm's producer does, and the consumer only waits for arrival.
// Reports per-SM bytes/clk and the loop time versus grid size, to tell a
// per-SM ingress limit from a chip-wide (L2) one.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/tma_bench tools/tma_bench.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

typedef unsigned int u32;
typedef unsigned long long u64;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ u64 gtimer() { u64 t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__global__ void __launch_bounds__(64, 1) tma_ingress(const __grid_constant__ CUtensorMap ma,
                                                     const __grid_constant__ CUtensorMap mb, int a_rows,
                                                     int b_rows, int K, int bk, int stages, int row_tiles,
                                                     u64* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) u64 full[16];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    const int stage_bytes = (a_rows + b_rows) * bk * 2;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(&ma) : "memory");
        asm volatile("prefetch.tensormap [%0];" :: "l"(&mb) : "memory");
    }
    __syncthreads();
    const int arow0 = (blockIdx.x % row_tiles) * a_rows;
    const int brow0 = (blockIdx.x / row_tiles) * b_rows;
    const int nkb = K / bk;
    u64 c0 = clock64(), t0 = gtimer();
    if (threadIdx.x == 0) {
        for (int i = 0; i < nkb + stages; ++i) {
            if (i >= stages) {      // consume stage (i - stages): wait for its bytes
                const int s = (i - stages) % stages;
                const u32 par = ((i - stages) / stages) & 1;
                asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                             :: "r"(smem_u32(&full[s])), "r"(par) : "memory");
            }
            if (i < nkb) {
                const int s = i % stages;
                const u32 bar = smem_u32(&full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(stage_bytes) : "memory");
                const u32 a_dst = smem_u32(smem + s * stage_bytes);
                const u32 b_dst = a_dst + a_rows * bk * 2;
                for (int ka = 0; ka < bk / 64; ++ka) {
                    const int kc = i * bk + ka * 64;
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                                 :: "r"(a_dst + ka * a_rows * 128), "l"(&ma), "r"(bar), "r"(kc), "r"(arow0) : "memory");
                    if (b_rows > 0)
                        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                                     :: "r"(b_dst + ka * b_rows * 128), "l"(&mb), "r"(bar), "r"(kc), "r"(brow0) : "memory");
                }
            }
        }
    }
    __syncthreads();
    u64 c1 = clock64(), t1 = gtimer();
    if (threadIdx.x == 0) {
        out[blockIdx.x * 2] = c1 - c0;
        out[blockIdx.x * 2 + 1] = t1 - t0;
    }
}

// Same loads, one box per operand per stage: 3-D maps {64, rows, K/64}
// (strides: K*2 bytes per row, 128 bytes per 64-element K atom) with box
// {64, rows, bk/64} land the stage's K atoms atom-major in one instruction.
__global__ void __launch_bounds__(64, 1) tma_ingress3d(const __grid_constant__ CUtensorMap ma,
                                                       const __grid_constant__ CUtensorMap mb, int a_rows,
                                                       int b_rows, int K, int bk, int stages, int row_tiles,
                                                       u64* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) u64 full[16];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    const int stage_bytes = (a_rows + b_rows) * bk * 2;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int arow0 = (blockIdx.x % row_tiles) * a_rows;
    const int brow0 = (blockIdx.x / row_tiles) * b_rows;
    const int nkb = K / bk;
    u64 c0 = clock64(), t0 = gtimer();
    if (threadIdx.x == 0) {
        for (int i = 0; i < nkb + stages; ++i) {
            if (i >= stages) {
                const int s = (i - stages) % stages;
                const u32 par = ((i - stages) / stages) & 1;
                asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                             :: "r"(smem_u32(&full[s])), "r"(par) : "memory");
            }
            if (i < nkb) {
                const int s = i % stages;
                const u32 bar = smem_u32(&full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(stage_bytes) : "memory");
                const u32 a_dst = smem_u32(smem + s * stage_bytes);
                const u32 b_dst = a_dst + a_rows * bk * 2;
                const int katom = i * bk / 64;
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                             :: "r"(a_dst), "l"(&ma), "r"(bar), "r"(0), "r"(arow0), "r"(katom) : "memory");
                if (b_rows > 0)
                    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                                 :: "r"(b_dst), "l"(&mb), "r"(bar), "r"(0), "r"(brow0), "r"(katom) : "memory");
            }
        }
    }
    __syncthreads();
    u64 c1 = clock64(), t1 = gtimer();
    if (threadIdx.x == 0) {
        out[blockIdx.x * 2] = c1 - c0;
        out[blockIdx.x * 2 + 1] = t1 - t0;
    }
}

static CUtensorMap make_map3(void* base, int rows, int K, int box_rows, int box_atoms) {
    CUtensorMap m;
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(K / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)box_atoms};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode3 failed %d\n", (int)r); exit(1); }
    return m;
}

// Conv-like activation loads: a 4-D NHWC map {C=64, W, H, N} with box
// {64, tw, th, tn} (128 pixels x 128 B), shifted per filter tap like the
// implicit-GEMM producer; `taps` boxes per tile, tiles walked like the
// persistent conv kernel.
__global__ void __launch_bounds__(64, 1) tma_conv4d(const __grid_constant__ CUtensorMap mx, int tw, int th, int tn,
                                                    int W, int H, int N, int tiles_per_cta, int stages, u64* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) u64 full[16];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    const int stage_bytes = 128 * 128;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int wt = W / tw, ht = H / th;
    const int n_it = tiles_per_cta * 9;
    u64 c0 = clock64(), t0 = gtimer();
    if (threadIdx.x == 0) {
        for (int i = 0; i < n_it + stages; ++i) {
            if (i >= stages) {
                const int s = (i - stages) % stages;
                const u32 par = ((i - stages) / stages) & 1;
                asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                             :: "r"(smem_u32(&full[s])), "r"(par) : "memory");
            }
            if (i < n_it) {
                const int s = i % stages;
                const u32 bar = smem_u32(&full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(stage_bytes) : "memory");
                const int tile = blockIdx.x + (i / 9) * gridDim.x, tap = i % 9;
                const int w0 = (tile % wt) * tw, h0 = ((tile / wt) % ht) * th, n0 = (tile / (wt * ht)) * tn;
                const int dj = tap % 3 - 1, di = tap / 3 - 1;
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                             :: "r"(smem_u32(smem + s * stage_bytes)), "l"(&mx), "r"(bar), "r"(0), "r"(w0 + dj),
                                "r"(h0 + di), "r"(n0 % N) : "memory");
            }
        }
    }
    __syncthreads();
    u64 c1 = clock64(), t1 = gtimer();
    if (threadIdx.x == 0) {
        out[blockIdx.x * 2] = c1 - c0;
        out[blockIdx.x * 2 + 1] = t1 - t0;
    }
}

// Conv activation loads in TMA im2col mode: a run of `pixels` consecutive
// output pixels (linear over N x H x W), 64 channels each, one instruction
// per filter tap (the tap is the im2col offset).
__global__ void __launch_bounds__(64, 1) tma_conv_im2col(const __grid_constant__ CUtensorMap mx, int pixels, int W,
                                                         int H, int N, int tiles_per_cta, int stages, u64* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) u64 full[16];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    const int stage_bytes = pixels * 128;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int n_it = tiles_per_cta * 9;
    u64 c0 = clock64(), t0 = gtimer();
    if (threadIdx.x == 0) {
        for (int i = 0; i < n_it + stages; ++i) {
            if (i >= stages) {
                const int s = (i - stages) % stages;
                const u32 par = ((i - stages) / stages) & 1;
                asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                             :: "r"(smem_u32(&full[s])), "r"(par) : "memory");
            }
            if (i < n_it) {
                const int s = i % stages;
                const u32 bar = smem_u32(&full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(stage_bytes) : "memory");
                const int tile = blockIdx.x + (i / 9) * gridDim.x, tap = i % 9;
                const int m0 = (tile * pixels) % (N * H * W);
                const int q0 = m0 % W, p0 = (m0 / W) % H, n0 = m0 / (W * H);
                const unsigned short ow = (unsigned short)(tap % 3), oh = (unsigned short)(tap / 3);
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};"
                             :: "r"(smem_u32(smem + s * stage_bytes)), "l"(&mx), "r"(bar), "r"(0), "r"(q0 - 1),
                                "r"(p0 - 1), "r"(n0), "h"(ow), "h"(oh) : "memory");
            }
        }
    }
    __syncthreads();
    u64 c1 = clock64(), t1 = gtimer();
    if (threadIdx.x == 0) {
        out[blockIdx.x * 2] = c1 - c0;
        out[blockIdx.x * 2 + 1] = t1 - t0;
    }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static CUtensorMap make_map(void* base, int rows, int K, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
    return m;
}

int main() {
    const int N = 1024, K = 1024;
    void *a, *b;
    CK(cudaMalloc(&a, (size_t)N * K * 2));
    CK(cudaMalloc(&b, (size_t)N * K * 2));
    CK(cudaMemset(a, 0, (size_t)N * K * 2));
    CK(cudaMemset(b, 0, (size_t)N * K * 2));
    u64* d_out;
    CK(cudaMalloc(&d_out, sizeof(u64) * 2 * 1024));
    CK(cudaFuncSetAttribute(tma_ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    struct Cfg { int a_rows, b_rows, bk, stages; } cfgs[] = {
        {128, 64, 128, 3}, {128, 64, 128, 4}, {128, 64, 64, 6}, {128, 128, 128, 3}, {128, 32, 128, 4},
        {128, 32, 256, 2}, {256, 0, 128, 3}, {128, 0, 128, 4}, {128, 0, 256, 3}};
    CK(cudaFuncSetAttribute(tma_ingress3d, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    for (int mode = 0; mode < 2; ++mode)
    for (auto c : cfgs) {
        if (mode == 1 && c.b_rows == 0) continue;
        CUtensorMap ma = make_map(a, N, K, c.a_rows);
        CUtensorMap mb = make_map(b, N, K, c.b_rows > 0 ? c.b_rows : 8);
        const int row_tiles = N / c.a_rows;
        const int smem = (c.a_rows + c.b_rows) * c.bk * 2 * c.stages + 1024;
        for (int grid : {1, 128}) {
            CUtensorMap ma3 = make_map3(a, N, K, c.a_rows, c.bk / 64);
            CUtensorMap mb3 = make_map3(b, N, K, c.b_rows > 0 ? c.b_rows : 8, c.bk / 64);
            for (int rep = 0; rep < 3; ++rep) {
                if (mode == 0)
                    tma_ingress<<<grid, 64, smem>>>(ma, mb, c.a_rows, c.b_rows, K, c.bk, c.stages, row_tiles, d_out);
                else
                    tma_ingress3d<<<grid, 64, smem>>>(ma3, mb3, c.a_rows, c.b_rows, K, c.bk, c.stages, row_tiles, d_out);
            }
            CK(cudaDeviceSynchronize());
            u64 h[2 * 148];
            CK(cudaMemcpy(h, d_out, sizeof(u64) * 2 * grid, cudaMemcpyDeviceToHost));
            double cyc = 0, ns = 0, mx = 0;
            for (int i = 0; i < grid; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; if (h[2 * i + 1] > mx) mx = h[2 * i + 1]; }
            cyc /= grid; ns /= grid;
            const double bytes = (double)(c.a_rows + c.b_rows) * K * 2;
            printf(mode ? "3D " : "2D ");
            printf("tile A%3d+B%3d BK%3d st%d grid=%3d: %6.1f B/clk/SM  %6.1f GB/s/SM  loop %.2f us (slowest %.2f)  chip %.1f TB/s\n",
                   c.a_rows, c.b_rows, c.bk, c.stages, grid, bytes / cyc, bytes / ns, ns / 1e3, mx / 1e3,
                   grid * bytes / mx / 1e3);
        }
    }
    {
        // conv activations NHWC 32x56x56x64 bf16
        const int N = 32, H = 56, W = 56, C = 64;
        void* x;
        CK(cudaMalloc(&x, (size_t)N * H * W * C * 2));
        CK(cudaMemset(x, 0, (size_t)N * H * W * C * 2));
        CK(cudaFuncSetAttribute(tma_conv4d, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        int shapes[][3] = {{8, 8, 2}, {8, 4, 4}, {4, 8, 4}, {8, 2, 8}, {2, 8, 8}, {8, 1, 16}};
        for (auto& sh : shapes) {
            CUtensorMap m;
            cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
            cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * W * 2, (cuuint64_t)C * W * H * 2};
            cuuint32_t box[4] = {64, (cuuint32_t)sh[0], (cuuint32_t)sh[1], (cuuint32_t)sh[2]};
            cuuint32_t es[4] = {1, 1, 1, 1};
            CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, strides, box, es,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { printf("encode4 failed %d\n", (int)r); continue; }
            for (int stages : {4, 8}) {
                const int grid = 148, tiles = 5;
                for (int rep = 0; rep < 3; ++rep)
                    tma_conv4d<<<grid, 64, stages * 16384 + 1024>>>(m, sh[0], sh[1], sh[2], W, H, N, tiles, stages, d_out);
                CK(cudaDeviceSynchronize());
                u64 h[2 * 148];
                CK(cudaMemcpy(h, d_out, sizeof(u64) * 2 * grid, cudaMemcpyDeviceToHost));
                double ns = 0, cyc = 0;
                for (int i = 0; i < grid; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; }
                cyc /= grid; ns /= grid;
                const double bytes = tiles * 9.0 * 16384;
                printf("conv4d box w%d h%d n%d st%d: %6.1f B/clk/SM %6.1f GB/s/SM  %.0f ns per box\n", sh[0], sh[1], sh[2],
                       stages, bytes / cyc, bytes / ns, ns / (tiles * 9));
            }
        }
    }
    {
        const int N = 32, H = 56, W = 56, C = 64;
        void* x;
        CK(cudaMalloc(&x, (size_t)N * H * W * C * 2));
        CK(cudaMemset(x, 0, (size_t)N * H * W * C * 2));
        CK(cudaFuncSetAttribute(tma_conv_im2col, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        for (int pixels : {128, 256}) {
            CUtensorMap m;
            cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
            cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * W * 2, (cuuint64_t)C * W * H * 2};
            int lo[2] = {-1, -1}, hi[2] = {-1, -1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            CUresult r = cuTensorMapEncodeIm2col(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, strides, lo, hi, 64,
                                                 (cuuint32_t)pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { printf("encode im2col failed %d\n", (int)r); continue; }
            for (int stages : {4, 8}) {
                const int grid = 148, tiles = 5;
                for (int rep = 0; rep < 3; ++rep)
                    tma_conv_im2col<<<grid, 64, stages * pixels * 128 + 1024>>>(m, pixels, W, H, N, tiles, stages, d_out);
                CK(cudaDeviceSynchronize());
                u64 h[2 * 148];
                CK(cudaMemcpy(h, d_out, sizeof(u64) * 2 * grid, cudaMemcpyDeviceToHost));
                double ns = 0, cyc = 0;
                for (int i = 0; i < grid; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; }
                cyc /= grid; ns /= grid;
                const double bytes = tiles * 9.0 * pixels * 128;
                printf("im2col pixels %d st%d: %6.1f B/clk/SM %6.1f GB/s/SM  %.0f ns per box\n", pixels, stages,
                       bytes / cyc, bytes / ns, ns / (tiles * 9));
            }
        }
    }
    return 0;
}
