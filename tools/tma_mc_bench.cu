// TMA ingress microbenchmark for the multicast question (not product code).
// Each CTA streams an A tile (a_rows x K) and a B tile (b_rows x K) of
// L2-resident bf16 matrices through a ring of `stages` stages of BK columns
// and its consumer only waits for arrival -- the GEMM mainloop's loads with
// no MMA.  Layouts of one operand stage in shared memory:
//   atom-major  [K/64 atoms][rows][128 B]  one 3-D box {64, rows, BK/64}
//               (what opevo_gemm's fused-K producer lands today)
//   group-major [rows/8 groups][BK/64 atoms][8 rows][128 B]  one 4-D box
//               {64, 8, BK/64, rows/8}: a row slice is a contiguous range of
//               groups, so a cluster can split the A tile by rows and
//               multicast each slice into every CTA with one box; the UMMA
//               descriptor reads it with SBO = atoms * 1024 B.
// Modes: 0 atom-major; 1 group-major; 2 group-major with the A tile shared by
// a cluster of `csz` CTAs (each fetches a_rows/csz rows, .multicast::cluster
// to all), slots released cluster-wide (every consumer arrives on every
// producer's empty barrier) as a real multicast pipeline must.
// Reports received bytes per SM per clock, loop time, chip-wide rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/tma_mc_bench tools/tma_mc_bench.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

typedef unsigned int u32;
typedef unsigned long long u64;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ u64 gtimer() { u64 t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ u32 crank() { u32 r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void wait_bar(u32 bar, u32 par) {
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                 :: "r"(bar), "r"(par) : "memory");
}

__global__ void __launch_bounds__(64, 1) tma_mc(const __grid_constant__ CUtensorMap ma,
                                                const __grid_constant__ CUtensorMap mb, int mode, int a_rows,
                                                int b_rows, int K, int bk, int stages, int csz, u64* out) {
    // (slot release: relaxed remote arrives -- nothing is read from the
    // slots here; a real pipeline releases with tcgen05.commit's multicast
    // arrive, which needs no cluster-scope fence either)
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) u64 full[16];
    __shared__ __align__(8) u64 empty[16];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    const int stage_bytes = (a_rows + b_rows) * bk * 2;
    const u32 rank = (mode == 2) ? crank() : 0u;
    const int cl = (mode == 2) ? csz : 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&empty[s])), "r"(cl));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (mode == 2) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    // tiles: the cluster (or CTA) shares one A row tile; B tiles per CTA
    const int row_tiles = 1024 / a_rows;
    const int unit = (int)blockIdx.x / cl;
    const int arow0 = (unit % row_tiles) * a_rows;
    const int brow0 = (((int)blockIdx.x / row_tiles) * b_rows) % 1024;
    const int nkb = K / bk;
    const int atoms = bk / 64;
    const int a_slice = a_rows / cl;          // rows this CTA fetches (mode 2)
    u64 c0 = clock64(), t0 = gtimer();
    if (threadIdx.x == 0) {
        for (int i = 0; i < nkb; ++i) {
            const int s = i % stages;
            const u32 ph = (i / stages) & 1;
            if (i >= stages) wait_bar(smem_u32(&empty[s]), ph ^ 1);
            const u32 bar = smem_u32(&full[s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(stage_bytes) : "memory");
            const u32 a_dst = smem_u32(smem + s * stage_bytes);
            const u32 b_dst = a_dst + a_rows * bk * 2;
            if (mode == 0) {
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                             :: "r"(a_dst), "l"(&ma), "r"(bar), "r"(0), "r"(arow0), "r"(i * atoms) : "memory");
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                             :: "r"(b_dst), "l"(&mb), "r"(bar), "r"(0), "r"(brow0), "r"(i * atoms) : "memory");
            } else if (mode == 1) {
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                             :: "r"(a_dst), "l"(&ma), "r"(bar), "r"(0), "r"(0), "r"(i * atoms), "r"(arow0 / 8) : "memory");
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                             :: "r"(b_dst), "l"(&mb), "r"(bar), "r"(0), "r"(0), "r"(i * atoms), "r"(brow0 / 8) : "memory");
            } else {
                // my slice of the shared A tile, into every CTA of the cluster
                const u32 a_off = a_dst + rank * (a_slice / 8) * atoms * 1024;
                const unsigned short mask = (unsigned short)((1u << cl) - 1);
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                             " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;"
                             :: "r"(a_off), "l"(&ma), "r"(bar), "r"(0), "r"(0), "r"(i * atoms),
                                "r"((arow0 + (int)rank * a_slice) / 8), "h"(mask) : "memory");
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                             :: "r"(b_dst), "l"(&mb), "r"(bar), "r"(0), "r"(0), "r"(i * atoms), "r"(brow0 / 8) : "memory");
            }
        }
    } else if (threadIdx.x == 32) {
        // consumer: wait for each stage, release it (cluster-wide in mode 2)
        for (int i = 0; i < nkb; ++i) {
            const int s = i % stages;
            wait_bar(smem_u32(&full[s]), (i / stages) & 1);
            if (mode == 2) {
                for (int r = 0; r < cl; ++r) {
                    u32 remote;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&empty[s])), "r"(r));
                    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" :: "r"(remote) : "memory");
                }
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
            }
        }
    }
    __syncthreads();
    u64 c1 = clock64(), t1 = gtimer();
    if (mode == 2) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) {
        out[blockIdx.x * 2] = c1 - c0;
        out[blockIdx.x * 2 + 1] = t1 - t0;
    }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static CUtensorMap map3(void* base, int rows, int K, int box_rows, int box_atoms) {
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

// group-major view {64, 8, K/64, rows/8}: strides row K*2, atom 128, group 8*K*2
static CUtensorMap map4(void* base, int rows, int K, int box_rows, int box_atoms) {
    CUtensorMap m;
    cuuint64_t dims[4] = {64, 8, (cuuint64_t)(K / 64), (cuuint64_t)(rows / 8)};
    cuuint64_t strides[3] = {(cuuint64_t)K * 2, 128, (cuuint64_t)K * 16};
    cuuint32_t box[4] = {64, 8, (cuuint32_t)box_atoms, (cuuint32_t)(box_rows / 8)};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode4 failed %d (box rows %d atoms %d)\n", (int)r, box_rows, box_atoms); exit(1); }
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
    CK(cudaFuncSetAttribute(tma_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(tma_mc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    struct Cfg { int a_rows, b_rows, bk, stages; } cfgs[] = {
        {128, 64, 128, 4}, {128, 64, 64, 6}, {128, 64, 256, 2}, {128, 32, 128, 4}, {128, 128, 128, 3}};
    for (auto& c : cfgs) {
        for (int mode = 0; mode < 3; ++mode) {
            for (int gc : {1001, 1032, 1064, 1128, 1148, 2, 4, 8}) {
                const int csz = gc > 1000 ? 1 : gc;
                const int grid = gc > 1000 ? gc - 1000 : 128;
                if ((mode < 2) != (csz == 1)) continue;
                if (mode < 2 && grid != 128 && &c != &cfgs[0]) continue;
                if (mode == 2 && (c.a_rows / csz) % 8) continue;
                CUtensorMap ma = mode == 0 ? map3(a, N, K, c.a_rows, c.bk / 64)
                                           : map4(a, N, K, mode == 2 ? c.a_rows / csz : c.a_rows, c.bk / 64);
                CUtensorMap mb = mode == 0 ? map3(b, N, K, c.b_rows, c.bk / 64) : map4(b, N, K, c.b_rows, c.bk / 64);
                const int smem = (c.a_rows + c.b_rows) * c.bk * 2 * c.stages + 1024;
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(64);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = (mode == 2) ? csz : 1;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                for (int rep = 0; rep < 5; ++rep)
                    CK(cudaLaunchKernelEx(&cfg, tma_mc, ma, mb, mode, c.a_rows, c.b_rows, K, c.bk, c.stages, csz, d_out));
                CK(cudaDeviceSynchronize());
                u64 h[2 * 148];
                CK(cudaMemcpy(h, d_out, sizeof(u64) * 2 * grid, cudaMemcpyDeviceToHost));
                double cyc = 0, ns = 0, mx = 0;
                for (int i = 0; i < grid; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; if (h[2 * i + 1] > mx) mx = h[2 * i + 1]; }
                cyc /= grid; ns /= grid;
                const double bytes = (double)(c.a_rows + c.b_rows) * K * 2;     // received per CTA
                const double issued = (double)((mode == 2 ? c.a_rows / csz : c.a_rows) + c.b_rows) * K * 2;
                printf("%-12s grid %3d csz %d  A%3d+B%3d BK%3d st%d: recv %6.1f B/clk/SM (issued %6.1f)  loop %.2f us (slowest %.2f)  chip recv %.1f TB/s\n",
                       mode == 0 ? "atom-major" : mode == 1 ? "group-major" : "group+mc", grid, csz, c.a_rows, c.b_rows,
                       c.bk, c.stages, bytes / cyc, issued / cyc, ns / 1e3, mx / 1e3, grid * bytes / mx / 1e3);
            }
        }
    }
    return 0;
}
