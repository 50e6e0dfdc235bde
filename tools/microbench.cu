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

template <int N, int M = 128>
__global__ void __launch_bounds__(128, 1) mma_bench(u64* out, int iters, int a_shift_rows, int b_off) {
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
    constexpr u32 IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((u32)(N >> 3) << 17) | ((u32)(M >> 4) << 24);
    constexpr u64 HI = ((u64)1 << 16) | ((u64)(1024 >> 4) << 32) | ((u64)1 << 46) | ((u64)2 << 61);
    // a_shift_rows: the A descriptor starts that many 128-byte rows into the
    // tile (the conv halo-line taps' shifted operands; 8 = one whole group)
    // b_off: byte offset of the B tile from the A tile (resident-panel placements)
    const u32 a0 = smem_u32(smem) + 128u * (u32)a_shift_rows, b0 = smem_u32(smem) + (u32)b_off;
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

// The conv halo-line MMA pattern without loads: per K block, KW = 3 taps x 4
// K16 steps, tap dj reading A at +dj rows and its own 64-row B tile (8 KB
// apart), N = 64, one accumulator; variants: flags bit 0 = A unshifted,
// bit 1 = one B tile for all taps, bit 2 = a tcgen05.commit after every K
// block (as the kernel releases its stages), bit 3 = B tiles 72 KB away
// (a resident weight panel), bit 4 = four "epilogue" warps streaming
// tcgen05.ld from another TMEM buffer meanwhile, bit 5 = those warps also
// write the loaded values to shared memory (the epilogue's staging), bit 6 =
// tcgen05.fence::after_thread_sync before every K block, bit 7 = a ring of
// `ring` stages: every K block commits to its stage's barrier and the MMA
// warp waits for that commit (the MMAs' completion) before reusing the stage
// -- the kernel's slot turnaround without the producer's relay.
__global__ void __launch_bounds__(256, 1) mma_halo_bench(u64* out, int iters, int flags, int ring,
                                                         int wait_kind) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    __shared__ u64 bar, cbar, rbar[8];
    __shared__ u32 tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) ((u32*)smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        mbar_init(smem_u32(&cbar), 1);
        for (int r = 0; r < 8; ++r) mbar_init(smem_u32(&rbar[r]), 1);
        if (flags & 128) {
            if (ring > 7) ring = 7;
            // rbar[7] completes phase 0 now (wait_kind 4 waits on it)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&rbar[7])) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = tslot;
    constexpr u32 IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((u32)(64 >> 3) << 17) | ((u32)(128 >> 4) << 24);
    if (warp >= 4 && (flags & 16)) {
        // "epilogue": loop over TMEM columns 64..127 of this warp's lane quarter
        const u32 q = (u32)(warp & 3);
        const u32 addr = tmem + 64u + ((q * 32u) << 16);
        float sink = 0.f;
        unsigned char* stg = smem + 150 * 1024 + (warp - 4) * 4096;
        while (!done) {
            u32 r[64];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                         "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,"
                         "%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,"
                         "%60,%61,%62,%63}, [%64];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                           "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                           "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                           "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                           "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]),
                           "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]),
                           "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
                           "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
                           "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]),
                           "=r"(r[63])
                         : "r"(addr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (flags & 32) {
                const int lane = threadIdx.x & 31;
#pragma unroll
                for (int j = 0; j < 64; j += 4)
                    *reinterpret_cast<uint4*>(stg + ((lane * 16 + j / 4) % 256) * 16) = make_uint4(r[j], r[j + 1], r[j + 2], r[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 64; ++j) sink += __uint_as_float(r[j]);
            }
        }
        if (sink == 12345.f) out[1000] = 1;
    }
    constexpr u64 HI = ((u64)1 << 16) | ((u64)(1024 >> 4) << 32) | ((u64)1 << 46) | ((u64)2 << 61);
    const u32 a0 = smem_u32(smem);
    const u32 b0 = a0 + ((flags & 8) ? 96 * 1024 : 24 * 1024);
    if (warp == 0) {
        u64 t0 = 0, t1 = 0, c0 = 0, c1 = 0;
        for (int rep = 0; rep < 2; ++rep) {
            c0 = clock64(); t0 = gtimer();
            for (int i = 0; i < iters; ++i) {
                const int g = rep * iters + i;        // K blocks issued so far
                if ((flags & 128) && g >= ring && wait_kind < 8) {     // stage g % ring: wait for its previous use
                    const u32 rb = smem_u32(&rbar[g % ring]), par = ((g / ring) - 1) & 1;
                    if (wait_kind == 0) {
                        mbar_wait(rb, par);
                    } else if (wait_kind == 1) {      // test_wait spin (no suspend)
                        u32 ok = 0;
                        while (!ok)
                            asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; "
                                         "selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(rb), "r"(par) : "memory");
                    } else if (wait_kind == 4) {      // a barrier whose phase 0 completed at init
                        mbar_wait(smem_u32(&rbar[7]), 0);
                    } else if (wait_kind == 6) {      // no wait at all (commits only)
                    } else if (wait_kind == 5) {      // the real wait, every 4th K block only
                        if (g % 4 == 0) mbar_wait(rb, par);
                    } else {                          // try_wait with a suspend-time hint (ns)
                        u32 ok = 0;
                        while (!ok)
                            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; "
                                         "selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(rb), "r"(par), "r"(wait_kind == 2 ? 0u : 100u) : "memory");
                    }
                }
                if (flags & 64) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (wait_kind >= 1000) {
                    // a try_wait on an already-completed barrier (the kernel's
                    // full-barrier fast path), nothing else
                    u32 ok;
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                                 "selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(smem_u32(&rbar[7])), "r"(0u) : "memory");
                    if (!ok) out[998] = 1;
                } else if (wait_kind >= 8) {
                    // bookkeeping between K blocks: a chain of dependent integer ops
                    u32 x = (u32)g;
                    for (int q = 0; q < wait_kind - 8; ++q) asm volatile("mad.lo.u32 %0, %0, 3, 1;" : "+r"(x));
                    if (x == 0x12345u) out[999] = x;
                }
                for (int dj = 0; dj < 3; ++dj) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const u32 aoff = ((flags & 1) ? 0u : (u32)dj * 128u) + k * 32;
                        const u32 boff = ((flags & 2) ? 0u : (u32)dj * 8192u) + k * 32;
                        const u64 ad = HI | (u64)(((a0 + aoff) >> 4) & 0x3FFF);
                        const u64 bd = HI | (u64)(((b0 + boff) >> 4) & 0x3FFF);
                        const u32 acc = (i | dj | k) ? 1u : 0u;
                        asm volatile("{ .reg .pred e, p; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; "
                                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                                     :: "r"(tmem), "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
                    }
                }
                if (flags & 4)
                    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }"
                                 :: "r"(smem_u32(&cbar)) : "memory");
                if (flags & 128)
                    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }"
                                 :: "r"(smem_u32(&rbar[g % ring])) : "memory");
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
            done = 1;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(tmem));
}

// Issue-rate probe: 12 MMAs (3 taps x 4 K16, N = 64) per K block from
// ONE asm block -- one elect, descriptors = 2 base registers + immediate
// offsets inside the block -- vs the per-MMA asm blocks above.
__global__ void __launch_bounds__(128, 1) mma_block12_bench(u64* out, int iters) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    __shared__ u64 bar;
    __shared__ u32 tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((u32*)smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
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
    constexpr u64 HI = ((u64)1 << 16) | ((u64)(1024 >> 4) << 32) | ((u64)1 << 46) | ((u64)2 << 61);
    const u64 ad = HI | (u64)((smem_u32(smem) >> 4) & 0x3FFF);
    const u64 bd = HI | (u64)(((smem_u32(smem) + 24 * 1024) >> 4) & 0x3FFF);
    if (warp == 0) {
        u64 t0 = 0, t1 = 0, c0 = 0, c1 = 0;
        for (int rep = 0; rep < 2; ++rep) {
            c0 = clock64(); t0 = gtimer();
            for (int i = 0; i < iters; ++i) {
                // A: tap dj at +dj rows (8 x 16-byte units), K16 at +2; B: tap at +8 KB (512), K16 at +2
#define MMA12_ONE(DA, DB) "add.s64 a, %1, " #DA "; add.s64 b, %2, " #DB "; @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t; "
                asm volatile("{ .reg .pred e, t; .reg .b64 a, b; elect.sync _|e, 0xffffffff; setp.ne.b32 t, %4, 0; "
                             MMA12_ONE(0, 0) MMA12_ONE(2, 2) MMA12_ONE(4, 4) MMA12_ONE(6, 6)
                             MMA12_ONE(8, 512) MMA12_ONE(10, 514) MMA12_ONE(12, 516) MMA12_ONE(14, 518)
                             MMA12_ONE(16, 1024) MMA12_ONE(18, 1026) MMA12_ONE(20, 1028) MMA12_ONE(22, 1030) "}"
                             :: "r"(tmem), "l"(ad), "l"(bd), "r"(IDESC), "r"(i | rep));
#undef MMA12_ONE
            }
            asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }"
                         :: "r"(smem_u32(&bar)) : "memory");
            mbar_wait(smem_u32(&bar), rep & 1);
            c1 = clock64(); t1 = gtimer();
        }
        if (threadIdx.x == 0) {
            out[0] = c1 - c0;
            out[1] = t1 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tmem));
}

// the kernel's mbar_wait: a fast-path try_wait, then a spin with a
// %globaltimer watchdog (v = 4 uses it for the per-K-block full wait)
__device__ __forceinline__ void wd_wait(u32 bar, u32 parity) {
    u32 done;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                 "selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    if (done) return;
    const u64 t0 = gtimer();
    while (true) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                     "selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
        if (done) return;
        if (gtimer() - t0 > 4000000000ull) asm volatile("trap;");
    }
}

// Issue-cost probe in the kernel's loop shape: per K block a try_wait on a
// (completed) full barrier, 12 MMAs (3 taps x 4 K16, N = 64), a commit.
//   v = 0: per tap one asm block of 4 MMAs with 64-bit descriptor adds (the
//          kernel's umma1_atom<4>)
//   v = 1: ONE asm block per K block, one elect, descriptors rebuilt from
//          32-bit low words + a constant high word (mov.b64 {lo, hi})
//   v = 2 / 3: v0 plus a warp spinning on an mbarrier try_wait (+ %globaltimer
//          watchdog, as the kernel's waiting roles do) on the SAME SM
//          sub-partition as the MMA warp (warp 4) / on another one (warp 5)
__global__ void __launch_bounds__(256, 1) mma_issue_bench(u64* out, int iters, int v) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((u64)smem_raw + 1023) & ~1023ull);
    __shared__ u64 bar, cbar, fbar, never;
    __shared__ u32 tslot;
    __shared__ volatile int done;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((u32*)smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        done = 0;
        mbar_init(smem_u32(&never), 1);
        mbar_init(smem_u32(&bar), 1);
        mbar_init(smem_u32(&cbar), 1);
        mbar_init(smem_u32(&fbar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&fbar)) : "memory");
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
    constexpr u64 HI = ((u64)1 << 16) | ((u64)(1024 >> 4) << 32) | ((u64)1 << 46) | ((u64)2 << 61);
    const u32 alo = (u32)(HI | (u64)((smem_u32(smem) >> 4) & 0x3FFF));
    const u32 blo = (u32)(HI | (u64)(((smem_u32(smem) + 16 * 1024) >> 4) & 0x3FFF));
    const u32 dhi = (u32)(HI >> 32);
    const u64 ad = ((u64)dhi << 32) | alo, bd = ((u64)dhi << 32) | blo;
    if (v == 7 && warp == 4) {
        // a TMA-like writer: bulk copies (L2 -> this CTA's shared memory, 6 x 8 KB
        // in flight) into a scratch area while the MMA warp runs; the bytes
        // it landed are reported in out[600 + block]
        __shared__ __align__(8) u64 wb[6];
        const int lane = threadIdx.x & 31;
        if (lane == 0) {
            for (int q = 0; q < 6; ++q) mbar_init(smem_u32(&wb[q]), 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        u64 landed = 0;
        int it = 0;
        const char* src = reinterpret_cast<const char*>(out) + 8192;
        if (lane == 0) {
            for (int q = 0; q < 6; ++q) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&wb[q])), "r"(8192) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             :: "r"(smem_u32(smem + 48 * 1024 + q * 8192)), "l"(src), "r"(8192), "r"(smem_u32(&wb[q])) : "memory");
            }
            while (!done) {
                const int q = it % 6;
                mbar_wait(smem_u32(&wb[q]), (it / 6) & 1);
                landed += 8192;
                ++it;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&wb[q])), "r"(8192) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             :: "r"(smem_u32(smem + 48 * 1024 + q * 8192)), "l"(src), "r"(8192), "r"(smem_u32(&wb[q])) : "memory");
            }
            for (int r = 0; r < 6; ++r, ++it) mbar_wait(smem_u32(&wb[it % 6]), (it / 6) & 1);
            out[600 + blockIdx.x] = landed;
        }
        __syncwarp();
    }
    if ((v == 2 && warp == 4) || (v == 3 && warp == 5)) {
        while (!done) {
            u32 ok;
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                         "selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(smem_u32(&never)), "r"(0u) : "memory");
            if (ok || gtimer() == 0) out[997] = 1;
        }
    }
    if (warp == 0) {
        u64 c0 = 0, c1 = 0;
        for (int rep = 0; rep < 2; ++rep) {
            c0 = clock64();
            for (int i = 0; i < iters; ++i) {
                if (v == 4) {
                    wd_wait(smem_u32(&fbar), 0u);
                } else {
                    u32 ok;
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                                 "selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(smem_u32(&fbar)), "r"(0u) : "memory");
                    if (!ok) out[998] = 1;
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const u32 acc = (i | rep) ? 1u : 0u;
                // v = 5: the K blocks cycle through 4 stage slots 24 KB apart
                // (fresh shared memory for every K block, as in the kernel's ring)
                const u64 soff = (v == 5) ? (u64)((i & 3) * (24 * 1024 / 16)) : 0ull;
                if (v == 6) {
                    // one thread issues (no elect / predicate per MMA)
                    if ((threadIdx.x & 31) == 0) {
#pragma unroll
                        for (int dj = 0; dj < 3; ++dj) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const u64 a = ad + (u64)(dj * 8 + k * 2), b = bd + (u64)(dj * 512 + k * 2);
                                const u32 accd = (dj | k) ? 1u : acc;
                                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; "
                                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                                             :: "r"(tmem), "l"(a), "l"(b), "r"(IDESC), "r"(accd));
                            }
                        }
                    }
                    __syncwarp();
                } else if (v != 1) {
                    for (int dj = 0; dj < 3; ++dj) {
                        const u64 a = ad + soff + (u64)(dj * 8), b = bd + soff + (u64)(dj * 512);
                        asm volatile("{ .reg .pred e, p, t; .reg .b64 a1, b1, a2, b2, a3, b3; elect.sync _|e, 0xffffffff; "
                                     "setp.ne.b32 p, %4, 0; setp.eq.b32 t, 0, 0; "
                                     "add.s64 a1, %1, 2; add.s64 b1, %2, 2; add.s64 a2, %1, 4; add.s64 b2, %2, 4; "
                                     "add.s64 a3, %1, 6; add.s64 b3, %2, 6; "
                                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; "
                                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t; "
                                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t; "
                                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t; }"
                                     :: "r"(tmem), "l"(a), "l"(b), "r"(IDESC), "r"(dj == 0 ? acc : 1u));
                    }
                } else {
#define MI_ONE(DA, DB) "add.u32 al, %1, " #DA "; add.u32 bl, %2, " #DB "; mov.b64 a, {al, %5}; mov.b64 b, {bl, %5}; " \
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t; "
                    asm volatile("{ .reg .pred e, p, t; .reg .b32 al, bl; .reg .b64 a, b; elect.sync _|e, 0xffffffff; "
                                 "setp.ne.b32 p, %4, 0; setp.eq.b32 t, 0, 0; "
                                 "mov.b64 a, {%1, %5}; mov.b64 b, {%2, %5}; "
                                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, p; "
                                 MI_ONE(2, 2) MI_ONE(4, 4) MI_ONE(6, 6)
                                 MI_ONE(8, 512) MI_ONE(10, 514) MI_ONE(12, 516) MI_ONE(14, 518)
                                 MI_ONE(16, 1024) MI_ONE(18, 1026) MI_ONE(20, 1028) MI_ONE(22, 1030) "}"
                                 :: "r"(tmem), "r"(alo), "r"(blo), "r"(IDESC), "r"(acc), "r"(dhi));
#undef MI_ONE
                }
                if (v == 6) {
                    if ((threadIdx.x & 31) == 0)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                     :: "r"(smem_u32(&cbar)) : "memory");
                    __syncwarp();
                } else {
                    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }"
                                 :: "r"(smem_u32(&cbar)) : "memory");
                }
            }
            asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }"
                         :: "r"(smem_u32(&bar)) : "memory");
            mbar_wait(smem_u32(&bar), rep & 1);
            c1 = clock64();
        }
        if (threadIdx.x == 0) { out[blockIdx.x] = c1 - c0; done = 1; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tmem));
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

template <int N, int M = 128>
void run_mma(u64* d_out, int grid, int shift = 0, int b_off = 160 * 128) {
    const int smem = b_off + 256 * 64 * 2 + 1024;
    CK(cudaFuncSetAttribute(mma_bench<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int iters = 256;
    mma_bench<N, M><<<grid, 128, smem>>>(d_out, iters, shift, b_off);
    CK(cudaDeviceSynchronize());
    u64 h[2 * 148];
    CK(cudaMemcpy(h, d_out, sizeof(u64) * 2 * grid, cudaMemcpyDeviceToHost));
    double cyc = 0, ns = 0;
    for (int i = 0; i < grid; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; }
    cyc /= grid; ns /= grid;
    const int mmas = iters * 4;
    const double flop = 2.0 * M * N * 16 * mmas;
    printf("mma M=%d N=%3d grid=%3d A shift %d rows B at +%6d: %.1f cyc/MMA (ideal %d), %.2f GHz, %.2f TFLOP/s/SM -> %.0f TFLOP/s x148\n",
           M, N, grid, shift, b_off, cyc / mmas, M * N / 256, cyc / ns, flop / ns / 1e3, 148 * flop / ns / 1e3);
}

int main() {
    u64* d_out;
    CK(cudaMalloc(&d_out, sizeof(u64) * 2 * 1024));
    if (getenv("MMA_M64")) {      // M = 64 (e.g. conv with Cout as M and pixels as N)
        for (int g : {1, 148}) {
            run_mma<64, 64>(d_out, g);
            run_mma<128, 64>(d_out, g);
            run_mma<256, 64>(d_out, g);
            run_mma<64, 128>(d_out, g);
            run_mma<256, 128>(d_out, g);
        }
        for (int sh : {0, 1, 2, 8}) run_mma<256, 64>(d_out, 1, 0, 160 * 128 + 128 * sh);   // B (pixels) shifted
        return 0;
    }
    for (int g : {1, 148}) {
        run_mma<64>(d_out, g);
        run_mma<128>(d_out, g);
        run_mma<256>(d_out, g);
    }
    // shifted A operands (conv halo taps): rows 1, 2 misalign every 8-row core matrix
    for (int sh : {0, 1, 2, 3, 8, 16}) run_mma<64>(d_out, 1, sh);
    for (int sh : {0, 1, 2}) run_mma<128>(d_out, 1, sh);
    for (int bo : {16384, 20480, 32768, 65536, 98304, 131072, 163840, 180224}) run_mma<64>(d_out, 1, 1, bo);
    {
        const int smem = 200 * 1024 + 1024;
        CK(cudaFuncSetAttribute(mma_halo_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int fr : {0, 8 * 65536, 9 * 65536, 10 * 65536, 12 * 65536, 16 * 65536, 24 * 65536,
                       1000 * 65536 + 128 + 1 * 256}) {
            const int flags = fr & 255, ring = (fr >> 8) & 255, wk = fr >> 16;
            const int iters = 128;
            mma_halo_bench<<<1, 256, smem>>>(d_out, iters, flags, ring, wk);
            CK(cudaDeviceSynchronize());
            u64 h[2];
            CK(cudaMemcpy(h, d_out, sizeof(u64) * 2, cudaMemcpyDeviceToHost));
            printf("mma halo pattern N=64 ring %d chain %3d wait %s flags %3d (%s%s%s%s%s%s%s): %.1f cyc/MMA\n", ring, wk >= 8 && wk < 1000 ? wk - 8 : 0,
                   wk == 0 ? "try_wait" : wk == 1 ? "test_wait" : wk == 2 ? "try_wait hint 0" : wk == 3 ? "try_wait hint 100ns"
                   : wk == 4 ? "on a completed barrier" : wk == 5 ? "every 4th K block" : wk >= 1000 ? "try_wait on a completed barrier only" : wk >= 8 ? "none, bookkeeping chain" : "none", flags,
                   flags & 1 ? "A unshifted " : "", flags & 2 ? "one B " : "", flags & 4 ? "commit/Kblock " : "",
                   flags & 8 ? "B far " : "", flags & 16 ? "+TMEM loads " : "", flags & 32 ? "+smem staging " : "",
                   flags & 64 ? "fence/Kblock " : "",
                   (double)h[0] / (iters * 12));
        }
    }
    {
        const int smem = 64 * 1024 + 1024;
        CK(cudaFuncSetAttribute(mma_block12_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const int iters = 128;
        mma_block12_bench<<<1, 128, smem>>>(d_out, iters);
        CK(cudaDeviceSynchronize());
        u64 h[2];
        CK(cudaMemcpy(h, d_out, sizeof(u64) * 2, cudaMemcpyDeviceToHost));
        printf("mma 12 per asm block N=64: %.1f cyc/MMA\n", (double)h[0] / (iters * 12));
    }
    {
        // two CTAs per SM, each with its own MMA-issuing warp: does the SM's
        // tensor pipe take more N = 64 MMAs than one issuing warp feeds?
        const int smem = 100 * 1024;
        CK(cudaFuncSetAttribute(mma_issue_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int v : {0, 7})
        for (int grid : {1, 148, 296}) {
            const int iters = 256;
            mma_issue_bench<<<grid, 256, smem>>>(d_out, iters, v);
            CK(cudaDeviceSynchronize());
            u64 h[1024];
            CK(cudaMemcpy(h, d_out, sizeof(u64) * 1024, cudaMemcpyDeviceToHost));
            double cyc = 0, bytes = 0;
            for (int i = 0; i < grid; ++i) { cyc += (double)h[i]; bytes += (double)h[600 + i]; }
            cyc /= grid;
            bytes /= grid;
            printf("mma issue v%d, %d CTAs (%s): %.1f cyc/MMA per CTA -> %.1f cyc/MMA per SM%s", v, grid,
                   grid == 296 ? "2 per SM" : "1 per SM", cyc / (iters * 12),
                   cyc / (iters * 12) / (grid == 296 ? 2.0 : 1.0), v == 7 ? "" : "\n");
            if (v == 7)
                printf("; concurrent bulk writes %.1f B/clk per CTA (%.1f per SM)\n", bytes / cyc,
                       bytes / cyc * (grid == 296 ? 2.0 : 1.0));
        }
    }
    {
        const int smem = 100 * 1024;
        CK(cudaFuncSetAttribute(mma_issue_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int v : {0, 6}) {
            const int iters = 128;
            mma_issue_bench<<<1, 256, smem>>>(d_out, iters, v);
            CK(cudaDeviceSynchronize());
            u64 h[1];
            CK(cudaMemcpy(h, d_out, sizeof(u64), cudaMemcpyDeviceToHost));
            printf("mma issue v%d (%s): %.1f cyc/MMA\n", v,
                   v == 0 ? "per-tap asm blocks, 64-bit adds" : v == 1 ? "one asm block per K block, 32-bit adds"
                   : v == 2 ? "v0 + a spinning warp on the MMA warp's sub-partition"
                   : v == 3 ? "v0 + a spinning warp elsewhere" : v == 4 ? "v0 with the kernel's watchdog wait"
                   : v == 5 ? "v0 with the K blocks cycling through 4 stage slots" : "one thread issues, no elect",
                   (double)h[0] / (iters * 12));
        }
    }
    if (getenv("MMA_ONLY")) return 0;
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
