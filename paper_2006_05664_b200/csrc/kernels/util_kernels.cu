// Support kernels of libopevo (compiled AOT by nvcc for sm_100a, embedded in
// the .so): deterministic input generation, the independent SIMT fp32
// reference for each operator, output comparison, layout conversion and the
// L2 flush used by cold-cache timing.
//
// Inputs are U(-1, 1) from a counter-based hash, so the CPU oracle
// (oracle/opevo_oracle.c) regenerates bit-identical operands without copying
// them back:  u = splitmix64(seed * GOLDEN + i) >> 40  (24 bits),
// x = u * 2^-23 - 1 (exact in fp32), bf16 operands = RNE(x).

typedef unsigned int u32;
typedef unsigned long long u64;
typedef unsigned short u16;

__device__ __forceinline__ u64 mix64(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float hashed_uniform(u64 seed, u64 i) {
    const u64 h = mix64(seed * 0x9E3779B97F4A7C15ull + i);
    return (float)(h >> 40) * (1.0f / 8388608.0f) - 1.0f;
}

__device__ __forceinline__ u16 f32_to_bf16_rne(float f) {
    u32 b = __float_as_uint(f);
    b += 0x7FFFu + ((b >> 16) & 1u);
    return (u16)(b >> 16);
}

__device__ __forceinline__ float bf16_to_f32(u16 h) {
    return __uint_as_float(((u32)h) << 16);
}

extern "C" __global__ void opevo_fill_bf16(u16* out, u64 n, u64 seed) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = f32_to_bf16_rne(hashed_uniform(seed, i));
}

extern "C" __global__ void opevo_fill_f32(float* out, u64 n, u64 seed) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = hashed_uniform(seed, i);
}

extern "C" __global__ void opevo_fill_u8(unsigned char* out, u64 n, unsigned char v) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = v;
}

// ---------------------------------------------------------------------------
// Reference GEMM: R[b][r][c] = sum_k A[b][r][k] * B[b][c][k]  (fp32 FFMA,
// 64x64 tile per block, 4x4 outputs per thread, k ascending).  Deliberately
// shares nothing with the tensor-core path.
// in_f32 = 0: operands are bf16; 1: fp32.
extern "C" __global__ void __launch_bounds__(256)
opevo_ref_gemm(const void* __restrict__ A, const void* __restrict__ B, float* __restrict__ R,
               int rows, int cols, int depth, int in_f32) {
    __shared__ float sa[16][64 + 1];
    __shared__ float sb[16][64 + 1];
    const int b = blockIdx.z;
    const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
    const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
    const u64 a_off = (u64)b * rows * depth, b_off = (u64)b * cols * depth;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int k0 = 0; k0 < depth; k0 += 16) {
        for (int t = threadIdx.x; t < 64 * 16; t += 256) {
            const int rr = t / 16, kk = t % 16;
            const int gr = r0 + rr, gc = c0 + rr, gk = k0 + kk;
            float va = 0.0f, vb = 0.0f;
            if (gr < rows && gk < depth) {
                const u64 idx = a_off + (u64)gr * depth + gk;
                va = in_f32 ? ((const float*)A)[idx] : bf16_to_f32(((const u16*)A)[idx]);
            }
            if (gc < cols && gk < depth) {
                const u64 idx = b_off + (u64)gc * depth + gk;
                vb = in_f32 ? ((const float*)B)[idx] : bf16_to_f32(((const u16*)B)[idx]);
            }
            sa[kk][rr] = va;
            sb[kk][rr] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = sa[kk][tr * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = sb[kk][tc * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gr = r0 + tr * 4 + i;
        if (gr >= rows) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gc = c0 + tc * 4 + j;
            if (gc < cols) R[(u64)b * rows * cols + (u64)gr * cols + gc] = acc[i][j];
        }
    }
}

// The same reference for large operands: 128x128 tile per block, 8x8
// outputs per thread (rows tr + 16 i, columns tc + 16 j), k ascending -- every
// output is the same sequential fp32 FMA chain over k as opevo_ref_gemm's,
// so the two agree bit for bit; ~2.5x the throughput (the reference is
// recomputed whenever operands are uploaded, i.e. every end-to-end step).
template <int NT>   // 128 rows x NT columns per block, 8 x NT/16 outputs per thread
__device__ __forceinline__ void ref_gemm_tile(const void* __restrict__ A, const void* __restrict__ B,
                                              float* __restrict__ R, int rows, int cols, int depth, int in_f32) {
    constexpr int CJ = NT / 16;
    // k-major staging; a thread's 8 rows (and CJ columns) are contiguous, so
    // its operands of one k step are 16-byte shared loads
    // (rows padded by 4 floats: the transposing stores spread over banks,
    // and every row still starts 16-byte aligned)
    __shared__ __align__(16) float sa[16][128 + 4];
    __shared__ __align__(16) float sb[16][NT + 4];
    const int b = blockIdx.z;
    const int r0 = blockIdx.y * 128, c0 = blockIdx.x * NT;
    const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
    const u64 a_off = (u64)b * rows * depth, b_off = (u64)b * cols * depth;
    float acc[8][CJ];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) acc[i][j] = 0.0f;
    // 128 rows (NT columns) x 16 k per operand, k fastest; the next chunk's
    // global loads are issued into registers before the current chunk's FMAs
    float ra[8], rb[CJ];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int t = threadIdx.x + q * 256;
            const int gr = r0 + t / 16, gk = k0 + t % 16;
            float va = 0.0f;
            if (gr < rows && gk < depth) {
                const u64 idx = a_off + (u64)gr * depth + gk;
                va = in_f32 ? ((const float*)A)[idx] : bf16_to_f32(((const u16*)A)[idx]);
            }
            ra[q] = va;
        }
#pragma unroll
        for (int q = 0; q < CJ; ++q) {
            const int t = threadIdx.x + q * 256;
            const int gc = c0 + t / 16, gk = k0 + t % 16;
            float vb = 0.0f;
            if (gc < cols && gk < depth) {
                const u64 idx = b_off + (u64)gc * depth + gk;
                vb = in_f32 ? ((const float*)B)[idx] : bf16_to_f32(((const u16*)B)[idx]);
            }
            rb[q] = vb;
        }
    };
    fetch(0);
    for (int k0 = 0; k0 < depth; k0 += 16) {
#pragma unroll
        for (int q = 0; q < 8; ++q) sa[(threadIdx.x + q * 256) % 16][(threadIdx.x + q * 256) / 16] = ra[q];
#pragma unroll
        for (int q = 0; q < CJ; ++q) sb[(threadIdx.x + q * 256) % 16][(threadIdx.x + q * 256) / 16] = rb[q];
        __syncthreads();
        if (k0 + 16 < depth) fetch(k0 + 16);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float av[8], bv[CJ];
            const float4* pa = reinterpret_cast<const float4*>(&sa[kk][tr * 8]);
            const float4 a0 = pa[0], a1 = pa[1];
            av[0] = a0.x; av[1] = a0.y; av[2] = a0.z; av[3] = a0.w;
            av[4] = a1.x; av[5] = a1.y; av[6] = a1.z; av[7] = a1.w;
            const float4* pb = reinterpret_cast<const float4*>(&sb[kk][tc * CJ]);
#pragma unroll
            for (int j = 0; j < CJ / 4; ++j) {
                const float4 v = pb[j];
                bv[4 * j] = v.x; bv[4 * j + 1] = v.y; bv[4 * j + 2] = v.z; bv[4 * j + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < CJ; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int gr = r0 + tr * 8 + i;
        if (gr >= rows) continue;
#pragma unroll
        for (int j = 0; j < CJ; ++j) {
            const int gc = c0 + tc * CJ + j;
            if (gc < cols) R[(u64)b * rows * cols + (u64)gr * cols + gc] = acc[i][j];
        }
    }
}

extern "C" __global__ void __launch_bounds__(256)
opevo_ref_gemm128(const void* __restrict__ A, const void* __restrict__ B, float* __restrict__ R,
                  int rows, int cols, int depth, int in_f32) {
    ref_gemm_tile<128>(A, B, R, rows, cols, depth, in_f32);
}

// 128 x 64 tiles: twice the blocks, for outputs whose 128 x 128 grid would
// leave most SMs idle (1024^2: 64 blocks on 148 SMs)
extern "C" __global__ void __launch_bounds__(256)
opevo_ref_gemm128x64(const void* __restrict__ A, const void* __restrict__ B, float* __restrict__ R,
                     int rows, int cols, int depth, int in_f32) {
    ref_gemm_tile<64>(A, B, R, rows, cols, depth, in_f32);
}

// Reference direct convolution on the paper's layouts:
// X NCHW, W OIHW (bf16), output written NHWC fp32 (the implicit-GEMM output
// layout).  One thread per output element, reduction order (ci, kh, kw).
extern "C" __global__ void opevo_ref_conv(const u16* __restrict__ X, const u16* __restrict__ W,
                                          float* __restrict__ R, int N, int C, int H, int Wd,
                                          int K, int KH, int KW, int stride, int pad, int HO, int WO) {
    const u64 total = (u64)N * HO * WO * K;
    for (u64 o = blockIdx.x * (u64)blockDim.x + threadIdx.x; o < total; o += (u64)gridDim.x * blockDim.x) {
        const int k = (int)(o % K);
        u64 p = o / K;
        const int wo = (int)(p % WO); p /= WO;
        const int ho = (int)(p % HO);
        const int n = (int)(p / HO);
        float acc = 0.0f;
        for (int c = 0; c < C; ++c)
            for (int i = 0; i < KH; ++i) {
                const int h = ho * stride - pad + i;
                if (h < 0 || h >= H) continue;
                for (int j = 0; j < KW; ++j) {
                    const int w = wo * stride - pad + j;
                    if (w < 0 || w >= Wd) continue;
                    const float x = bf16_to_f32(X[(((u64)n * C + c) * H + h) * Wd + w]);
                    const float f = bf16_to_f32(W[(((u64)k * C + c) * KH + i) * KW + j]);
                    acc = fmaf(x, f, acc);
                }
            }
        R[o] = acc;
    }
}

// The same convolution as a tiled SIMT implicit GEMM: 128 output pixels x
// 64 output channels per block, 8 x 4 per thread, the reduction index
// q = (c, i, j) ascending in chunks of 16 staged through shared memory (the
// activation gather applies the padding), so every output is the same fmaf
// chain over (ci, kh, kw) as opevo_ref_conv's (a padded tap contributes
// fmaf(0, w, acc) = acc).  ~100x faster than one thread per output, which
// matters when new operands are uploaded every generation (bench.py e2e).
extern "C" __global__ void __launch_bounds__(256)
opevo_ref_conv_tiled(const u16* __restrict__ X, const u16* __restrict__ W, float* __restrict__ R, int N,
                     int C, int H, int Wd, int K, int KH, int KW, int stride, int pad, int HO, int WO) {
    __shared__ float sx[16][128 + 4];
    __shared__ float sw[16][64 + 4];
    const int P = N * HO * WO, Q = C * KH * KW;
    const int p0 = blockIdx.x * 128, k0 = blockIdx.y * 64;
    const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    // 128 pixels x 16 reduction steps (the activation gather applies the
    // padding) and 64 output channels x 16 steps (W rows are q-contiguous);
    // the next chunk is fetched into registers before the current one's FMAs
    float rx[8], rw[4];
    auto fetch = [&](int q0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int t = threadIdx.x + u * 256;
            const int p = p0 + t / 16, q = q0 + t % 16;
            float v = 0.0f;
            if (p < P && q < Q) {
                const int wo = p % WO, ho = (p / WO) % HO, n = p / (WO * HO);
                const int j = q % KW, i = (q / KW) % KH, c = q / (KW * KH);
                const int h = ho * stride - pad + i, w = wo * stride - pad + j;
                if (h >= 0 && h < H && w >= 0 && w < Wd)
                    v = bf16_to_f32(X[(((u64)n * C + c) * H + h) * Wd + w]);
            }
            rx[u] = v;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = threadIdx.x + u * 256;
            const int k = k0 + t / 16, q = q0 + t % 16;
            rw[u] = (k < K && q < Q) ? bf16_to_f32(W[(u64)k * Q + q]) : 0.0f;
        }
    };
    fetch(0);
    for (int q0 = 0; q0 < Q; q0 += 16) {
#pragma unroll
        for (int u = 0; u < 8; ++u) sx[(threadIdx.x + u * 256) % 16][(threadIdx.x + u * 256) / 16] = rx[u];
#pragma unroll
        for (int u = 0; u < 4; ++u) sw[(threadIdx.x + u * 256) % 16][(threadIdx.x + u * 256) / 16] = rw[u];
        __syncthreads();
        if (q0 + 16 < Q) fetch(q0 + 16);
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) {
            float xv[8], wv[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) xv[i] = sx[qq][tr + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) wv[j] = sw[qq][tc + 16 * j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xv[i], wv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int p = p0 + tr + 16 * i;
        if (p >= P) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = k0 + tc + 16 * j;
            if (k < K) R[(u64)p * K + k] = acc[i][j];
        }
    }
}

// NCHW -> NHWC (activations) and OIHW -> O(HW)I (weights: K-major rows).
extern "C" __global__ void opevo_nchw_to_nhwc(const u16* __restrict__ src, u16* __restrict__ dst,
                                              int N, int C, int H, int W) {
    const u64 total = (u64)N * C * H * W;
    for (u64 o = blockIdx.x * (u64)blockDim.x + threadIdx.x; o < total; o += (u64)gridDim.x * blockDim.x) {
        const int c = (int)(o % C);
        u64 p = o / C;
        const int w = (int)(p % W); p /= W;
        const int h = (int)(p % H);
        const int n = (int)(p / H);
        dst[o] = src[(((u64)n * C + c) * H + h) * W + w];
    }
}

// NCHW -> NHWC with the channels padded with zeros to Cp (dst has N*H*W*Cp
// elements): the conv kernels' layout, whose pixel rows must be >= 16 bytes
// and a whole UMMA K step (narrow Cin, e.g. 3 -> 16).  Also OIHW -> O(HW)I.
extern "C" __global__ void opevo_nchw_to_nhwc_pad(const u16* __restrict__ src, u16* __restrict__ dst,
                                                  int N, int C, int H, int W, int Cp) {
    const u64 total = (u64)N * Cp * H * W;
    for (u64 o = blockIdx.x * (u64)blockDim.x + threadIdx.x; o < total; o += (u64)gridDim.x * blockDim.x) {
        const int c = (int)(o % Cp);
        u64 p = o / Cp;
        const int w = (int)(p % W); p /= W;
        const int h = (int)(p % H);
        const int n = (int)(p / H);
        dst[o] = c < C ? src[(((u64)n * C + c) * H + h) * W + w] : (u16)0;
    }
}

// The inverse (padding dropped): an uploaded kernel-layout operand back to
// the paper layout the reference convolution reads.
extern "C" __global__ void opevo_nhwc_pad_to_nchw(const u16* __restrict__ src, u16* __restrict__ dst,
                                                  int N, int C, int H, int W, int Cp) {
    const u64 total = (u64)N * C * H * W;
    for (u64 o = blockIdx.x * (u64)blockDim.x + threadIdx.x; o < total; o += (u64)gridDim.x * blockDim.x) {
        const int w = (int)(o % W);
        u64 p = o / W;
        const int h = (int)(p % H); p /= H;
        const int c = (int)(p % C);
        const int n = (int)(p / C);
        dst[o] = src[(((u64)n * H + h) * W + w) * Cp + c];
    }
}

// ---------------------------------------------------------------------------
// out[0] = max |C - R|, out[1] = max |R|, out[2] = count of non-finite C.
// Non-negative floats compare like their bit patterns, so atomicMax on u32.
// Four outputs per step (16-byte R loads, 8- or 16-byte C loads), reduced in
// the warp, then in the block through shared memory: ONE set of atomics per
// block.  (One set per warp -- 32 K warps on the same two words for a
// 1024^2 output -- serialised at one L2 slice and cost ~0.1 ms per check.)
__device__ __forceinline__ void cmp_one(float c, float r, float& md, float& mr, u32& bad) {
    if (!isfinite(c)) { ++bad; return; }
    md = fmaxf(md, fabsf(c - r));
    mr = fmaxf(mr, fabsf(r));
}

extern "C" __global__ void __launch_bounds__(256) opevo_compare(const void* __restrict__ C,
                                                                const float* __restrict__ R, u64 n,
                                                                int c_f32, u32* __restrict__ out) {
    float md = 0.0f, mr = 0.0f;
    u32 bad = 0;
    const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    const u64 n4 = n / 4;
    for (u64 q = tid; q < n4; q += stride) {
        const float4 r = reinterpret_cast<const float4*>(R)[q];
        float c0, c1, c2, c3;
        if (c_f32) {
            const float4 c = reinterpret_cast<const float4*>(C)[q];
            c0 = c.x; c1 = c.y; c2 = c.z; c3 = c.w;
        } else {
            const uint2 u = reinterpret_cast<const uint2*>(C)[q];
            c0 = __uint_as_float(u.x << 16); c1 = __uint_as_float(u.x & 0xFFFF0000u);
            c2 = __uint_as_float(u.y << 16); c3 = __uint_as_float(u.y & 0xFFFF0000u);
        }
        cmp_one(c0, r.x, md, mr, bad);
        cmp_one(c1, r.y, md, mr, bad);
        cmp_one(c2, r.z, md, mr, bad);
        cmp_one(c3, r.w, md, mr, bad);
    }
    for (u64 i = 4 * n4 + tid; i < n; i += stride) {
        const float c = c_f32 ? ((const float*)C)[i] : bf16_to_f32(((const u16*)C)[i]);
        cmp_one(c, R[i], md, mr, bad);
    }
    for (int o = 16; o > 0; o >>= 1) {
        md = fmaxf(md, __shfl_xor_sync(0xffffffffu, md, o));
        mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    __shared__ float s_md[8], s_mr[8];
    __shared__ u32 s_bad[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { s_md[warp] = md; s_mr[warp] = mr; s_bad[warp] = bad; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            md = fmaxf(md, s_md[w]);
            mr = fmaxf(mr, s_mr[w]);
            bad += s_bad[w];
        }
        atomicMax(out + 0, __float_as_uint(md));
        atomicMax(out + 1, __float_as_uint(mr));
        if (bad) atomicAdd(out + 2, bad);
    }
}

// Streams a buffer larger than L2 so the next timed launch starts cold.
// A READ pass over a 2x-L2 buffer: every resident line is evicted (dirty
// ones -- the previous launch's output -- are written back now, during the
// flush) and L2 is left holding clean lines of this buffer, so the timed
// launch's misses cost no write-backs.  (A write pass would leave 126 MB of
// dirty lines whose write-back then shares HBM with the timed launch's
// reads: measured as half the HBM bandwidth for an HBM-bound operator.)
extern "C" __global__ void opevo_flush(uint4* buf, u64 n16, u32 salt) {
    uint4 acc = make_uint4(0u, 0u, 0u, 0u);
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n16; i += (u64)gridDim.x * blockDim.x) {
        const uint4 v = __ldcg(buf + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    // keeps the loads (never true in practice; the buffer is scratch anyway)
    if (acc.x == salt && acc.y == 0x9E3779B9u && acc.z == ~salt && acc.w == 0x7F4A7C15u) buf[0] = acc;
}

// Launch gate for timing: the stream stalls here while the host enqueues the
// timed launches, then the host writes `seq` into the mapped flag and the
// launches run back to back with no host gaps.  A %globaltimer timeout (the
// host never fails to open the gate, but a hung device would be a strike)
// releases the stream regardless.
extern "C" __global__ void opevo_gate(const u32* flag, u32 seq, u64 timeout_ns) {
    u64 t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        u32 v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if ((int)(v - seq) >= 0) return;
        u64 t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) return;
        __nanosleep(200);
    }
}
