// OpEvo B200 GEMM family (sm_100a): C = A . B^T, bf16 in, fp32 accumulate.
//
// JIT-instantiated by libopevo (NVRTC) once per canonical knob tuple; the
// knobs arrive as -D macros (see kernel_source.cpp / mapping.py):
//   OPEVO_BM      CTA rows: 64 (UMMA M=64), 128 (M=128), 256 (two M=128 atoms)
//   OPEVO_BN      CTA cols = UMMA N (16..256, multiple of 16)
//   OPEVO_BK      K elements staged per pipeline stage (16..256)
//   OPEVO_STAGES  depth of the TMA -> MMA shared-memory ring
//   OPEVO_BATCHED 1: 3-D tensor maps {K, rows, batch} (BatchMatMul)
//   OPEVO_OUT_F32 1: fp32 output (else bf16)
//   OPEVO_CLUSTER CTAs per cluster along the column-tile axis; the A tile is
//                 TMA-multicast to all of them (1 = no cluster)
//   OPEVO_CONV    1: implicit-GEMM Conv2d. A is the NHWC activation read by a
//                 4-D TMA box {C, TILE_W, TILE_H, TILE_N} shifted per filter
//                 tap; padding comes from TMA out-of-bounds zero fill.  B is
//                 the O(HW)I weight matrix [Cout][Kh*Kw*Cin].
//   OPEVO_TILE_H / OPEVO_TILE_W  conv output tile (BM = TILE_N*TILE_H*TILE_W)
//   OPEVO_HALO    KW > 0: conv "halo lines".  The tile is TILE_N*TILE_H lines of
//                 TILE_W = 17 - KW output pixels, each line padded to 16 tile
//                 rows (the last KW - 1 rows are junk and never stored).  One
//                 4-D box {C, 16, TILE_H, TILE_N} per filter row (di) holds the
//                 input pixels of all KW taps of that row: tap dj's A operand
//                 is the same box with the descriptor start moved dj rows (128 B;
//                 the SW128 pattern is keyed on the absolute shared address, so
//                 any whole-row shift stays canonical -- tools/swizzle_probe.cu).
//                 KW times fewer TMA boxes for (16 - TILE_W)/16 more MMA rows.
//   OPEVO_LINE    16 / 32: conv "padded lines" (any stride, no halo): the tile is
//                 TILE_N*TILE_H lines of TILE_W <= LINE output pixels, each
//                 line padded to LINE tile rows, one box per filter tap; the
//                 junk rows are computed and never stored.  Output widths
//                 that no power of two divides (27, 55, ...) tile this way.
//   OPEVO_CTA_GROUP 2: a cluster of two CTAs on neighbouring SMs computes a
//                 256 x BN tile with tcgen05.mma.cta_group::2 (M=256); each
//                 CTA stages 128 rows of A and BN/2 rows of B, so per-SM
//                 operand traffic (TMA ingress and smem reads) drops versus a
//                 single-CTA 256-row tile.  Only the leader CTA issues MMAs.
//                 Conv pairs: each CTA holds TILE_N images of the pair's
//                 2 x TILE_N (its own 128 tile rows).
//   Conv stride S: the activation tensor map traverses W and H with element
//                 stride S (box extents LINE*S / TILE_H*S input pixels land
//                 LINE / TILE_H output pixels' worth), so strided filters need
//                 no im2col buffer either.
//   OPEVO_SPLIT_CLUSTER S: split-K whose S slices of one tile run as one
//                 thread-block cluster.  After the mainloop each CTA stages
//                 its fp32 partial in shared memory and bulk-copies the row
//                 block owned by each peer into that peer's shared memory
//                 (cp.async.bulk shared::cluster, DSMEM); every CTA then sums
//                 its own row block in z order and writes it.  No partials
//                 touch global memory.
//   OPEVO_TF32X3  1: fp32 operands on the tensor cores, three kind::tf32 MMAs
//                 per K step (hi*hi + hi*lo + lo*hi, fp32-level accuracy).
//                 The host views each fp32 operand as bf16 pairs -- BK, depth
//                 and every byte offset keep the bf16 meaning, so K8 of tf32
//                 is one 32-byte K16 step -- and the epilogue warps write the
//                 lo part of each landed stage into a second area.
//   OPEVO_ACC     independent TMEM accumulators the K loop round-robins over
//                 (summed in the epilogue).  Consecutive MMAs into one
//                 accumulator form a dependent chain; for small N the chain
//                 latency, not the tensor-pipe rate, bounds the mainloop, and
//                 interleaving ACC chains hides it -- the tcgen05 analogue of
//                 the paper's virtual threads.
//
// Programmatic dependent launch: every CTA signals launch_dependents on entry
// and waits (griddepcontrol.wait) before its first global read/write, so a
// following launch overlaps its prologue (barrier init, TMEM alloc,
// descriptor prefetch) with this one's tail; the host sets the PDL launch
// attribute.
// Runtime: gridDim = (col tiles, row tiles, batch * split); split-K partials
// are reduced in-kernel by the last-arriving CTA of each tile (deterministic
// order z = 0..split-1).
//
// Layout: A [batch][rows][K], B [batch][cols][K] (both K-major, the natural
// UMMA operand order, "NT"), C [batch][rows][cols] row-major.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA
// issuer, warps 2..5 = epilogue (TMEM -> registers -> global).  Shared memory
// operands use the canonical K-major swizzled layout (SW128/64/32 by BK) that
// TMA writes and the UMMA descriptors read.
//
// The paper's thread-level tiling knobs have no tcgen05
// counterpart -- a single thread issues each MMA -- so they do not reach this
// file; see mapping.py for how a configuration becomes these macros.

#ifndef OPEVO_BM
#define OPEVO_BM 128
#endif
#ifndef OPEVO_BN
#define OPEVO_BN 128
#endif
#ifndef OPEVO_BK
#define OPEVO_BK 64
#endif
#ifndef OPEVO_STAGES
#define OPEVO_STAGES 4
#endif
#ifndef OPEVO_BATCHED
#define OPEVO_BATCHED 0
#endif
#ifndef OPEVO_OUT_F32
#define OPEVO_OUT_F32 0
#endif
#ifndef OPEVO_CLUSTER
#define OPEVO_CLUSTER 1
#endif
#ifndef OPEVO_CONV
#define OPEVO_CONV 0
#endif
#ifndef OPEVO_HALO
#define OPEVO_HALO 0       // conv: KW taps per halo box (0: one box per tap)
#endif
#ifndef OPEVO_LINE
#define OPEVO_LINE 0       // conv: padded lines of this many tile rows (0: dense tile)
#endif
#ifndef OPEVO_WBOX
#define OPEVO_WBOX 1       // halo lines: one 4-D weight box per filter row (0: per-tap 2-D boxes;
                           // experiments, with OPEVO_WBOX=0 in the host's environment too)
#endif
#ifndef OPEVO_X3_SMEM_ALO
#define OPEVO_X3_SMEM_ALO 0 // 1: 3xTF32 keeps A_lo in shared memory (the pre-X3T path; A/B)
#endif
#ifndef OPEVO_NARROW_EPI
#define OPEVO_NARROW_EPI 0 // 32-column epilogue staging (host rule: two CTAs per SM)
#endif
#ifndef OPEVO_TILE_H
#define OPEVO_TILE_H 1
#endif
#ifndef OPEVO_TILE_W
#define OPEVO_TILE_W 1
#endif
#ifndef OPEVO_CTA_GROUP
#define OPEVO_CTA_GROUP 1  // 2: CTA-pair MMA (cta_group::2, M=256 across two SMs)
#endif
#ifndef OPEVO_SPLIT_CLUSTER
#define OPEVO_SPLIT_CLUSTER 0  // S > 1: the S K-slices of a tile form a cluster and reduce via DSMEM
#endif
#ifndef OPEVO_B_RES
#define OPEVO_B_RES 0      // conv: the BN x K weight panel stays resident in shared memory
#endif
#ifndef OPEVO_SPLIT_TMA
#define OPEVO_SPLIT_TMA 0  // S > 1: split-K in one wave; slices 1..S-1 publish fp32 partials
                           // with TMA stores, slice 0 TMA-loads them and reduces
#endif
#ifndef OPEVO_BPU
#define OPEVO_BPU 1        // BatchMatMul: consecutive batches per work unit (one TMA box per
                           // operand and stage covers all of them; accumulators side by side)
#endif
#ifndef OPEVO_TF32X3
#define OPEVO_TF32X3 0     // fp32 GEMM as 3xTF32 on tcgen05 (fp32 in/out)
#endif
#ifndef OPEVO_ACC
#define OPEVO_ACC 1        // K-interleaved TMEM accumulators (1, 2, 4)
#endif
#ifndef OPEVO_ABLATE
#define OPEVO_ABLATE 0     // debug: 1 exit at entry, 2 no mainloop, 3 no TMA, 4 no MMA,
                           // 5 trap (fault injection: poisons the context), 6 no C stores,
                           // 7 no mainloop and no C stores
#endif
#ifndef OPEVO_TRACE
#define OPEVO_TRACE 0      // 1: per-CTA %globaltimer phase stamps into `ws` (debug)
#endif

#pragma nv_diag_suppress 177
typedef unsigned int u32;
typedef unsigned long long u64;
typedef unsigned short u16;

namespace opevo {

constexpr int BM = OPEVO_BM;
constexpr int BN = OPEVO_BN;
constexpr int BK = OPEVO_BK;
constexpr int STAGES = OPEVO_STAGES;
constexpr int CLUSTER = OPEVO_CLUSTER;
constexpr int CG = OPEVO_CTA_GROUP;

constexpr int SWZ = (BK * 2 >= 128) ? 128 : BK * 2;     // swizzle span in bytes
constexpr int ATOM_K = SWZ / 2;                          // K elements per swizzle row
constexpr int KATOMS = BK / ATOM_K;                      // swizzle atoms along K
constexpr int BM_CTA = (CG == 2) ? BM / 2 : BM;          // A rows resident in this CTA
constexpr int BN_LOAD = BN / CG;                          // B rows this CTA stages
constexpr int MATOMS = (BM_CTA == 256) ? 2 : 1;          // MMAs per k-step (M=128, or M=256 per pair)
constexpr int UMMA_M = (CG == 2) ? 256 : ((BM == 256) ? 128 : BM);
constexpr int BPU = OPEVO_BPU;
constexpr int A_SUB = BM_CTA * BK * 2;                    // one batch's A tile of a stage
constexpr int A_TILE = BPU * A_SUB;
constexpr int HKW = OPEVO_HALO;                          // conv taps served per halo box
constexpr bool HALO = HKW > 0;
constexpr bool B_RES = OPEVO_B_RES != 0;
constexpr int B_SUB = BN_LOAD * BK * 2;
constexpr int B_TILE = B_RES ? 0 : (HALO ? HKW : BPU) * B_SUB;   // per stage (0: panel resident)
constexpr bool X3 = OPEVO_TF32X3 != 0;
constexpr int LOAD_BYTES = A_TILE + B_TILE;               // what TMA lands per stage
constexpr int LO_OFF = LOAD_BYTES;                        // X3: lo parts, same layout
constexpr int STAGE_BYTES = X3 ? 2 * LOAD_BYTES : LOAD_BYTES;
constexpr int TX_BYTES = LOAD_BYTES * CG;                 // bytes landing per stage (pair)
constexpr int A_SLICE_ROWS = BM_CTA / CLUSTER;            // rows of A each cluster CTA fetches
// K-fused loads: with 128-byte swizzle the host encodes A and B as
// {64, rows, K/64 (, batch)} "atom" views (row stride K*2 bytes, atom stride
// 128 bytes), so one box {64, rows, KATOMS} lands a whole stage of an operand
// atom-major -- one TMA instruction per operand per stage instead of one per
// 64-wide K atom (per-instruction TMA cost, not bytes, bounds small stages).
// Multicast slices and conv taps keep per-atom boxes.
constexpr bool FUSED_K = (SWZ == 128) && (CLUSTER == 1) && !OPEVO_CONV;
constexpr int ACC = OPEVO_ACC;
constexpr int TMEM_USED = MATOMS * BN * ACC * BPU;
constexpr int TMEM_COLS = TMEM_USED <= 32 ? 32 : TMEM_USED <= 64 ? 64 :
                          TMEM_USED <= 128 ? 128 : TMEM_USED <= 256 ? 256 : 512;
constexpr u32 LAYOUT = SWZ == 128 ? 2u : SWZ == 64 ? 4u : 6u;
constexpr int EPI_COLS = (BN % 32 == 0) ? 32 : 16;    // split-K / DSMEM reduction chunks
// TMA-store epilogue chunk: 64 bf16 columns (one 128-byte swizzle row) when
// BN allows, so each chunk is one TMEM load, one proxy fence and one store
// (32 columns instead when the host's two-CTAs-per-SM rule asks for the
// smaller staging: OPEVO_NARROW_EPI, narrow_epi in opevo.cpp)
constexpr int STORE_COLS = (!OPEVO_OUT_F32 && BN % 64 == 0 && OPEVO_ACC == 1 && !OPEVO_NARROW_EPI) ? 64 : EPI_COLS;
constexpr int NUM_THREADS = 192;
constexpr int SMEM_ALIGN = 1024;
constexpr int TILE_H = OPEVO_TILE_H;
constexpr int TILE_W = OPEVO_TILE_W;
constexpr int LINE = OPEVO_LINE;
constexpr bool LINES = HALO || LINE > 0;                 // lines padded with junk rows
constexpr int LINE_ROWS = HALO ? 16 : (LINE > 0 ? LINE : TILE_W);   // tile rows per output line
constexpr int TILE_N = BM_CTA / (TILE_H * LINE_ROWS);     // images of this CTA's tile
constexpr int PAIR_TN = CG * TILE_N;                      // images of the (pair) tile
// padded lines may leave tile rows past TILE_N x TILE_H lines unloaded (junk,
// never stored): the activation box lands A_ROWS rows
constexpr int A_ROWS = OPEVO_CONV ? TILE_N * TILE_H * LINE_ROWS : BM_CTA;
constexpr int TX_STAGE = OPEVO_CONV ? (A_ROWS * BK * 2 + B_TILE) * CG : TX_BYTES;   // expect_tx per stage

static_assert(BM == 64 || BM == 128 || BM == 256 || (BM == 512 && CG == 2 && HKW > 0),
              "BM must be 64, 128 or 256 (512: a halo-line conv CTA pair, 256 rows per CTA)");
static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "BN must be a multiple of 16 in [16, 256]");
static_assert(BK % 16 == 0 && BK >= 16 && BK <= 256, "BK must be a multiple of 16 in [16, 256]");
static_assert(BK % ATOM_K == 0, "BK must tile the swizzle atom");
static_assert(TMEM_USED <= 512, "accumulator exceeds TMEM");
static_assert(ACC == 1 || ACC == 2 || ACC == 4, "ACC must be 1, 2 or 4");
static_assert((BK / 16) % ACC == 0, "each stage must feed every accumulator");
static_assert(BM % (8 * CLUSTER) == 0, "multicast slice must be whole 8-row groups");
static_assert(CG == 1 || (CG == 2 && (BM == 256 || BM == 512) && CLUSTER == 1 && BN % 16 == 0 &&
                           OPEVO_B_RES == 0),
              "CTA pairs: 256- (or halo 512-) row tiles, no extra multicast or resident weights");
static_assert(!HALO || (OPEVO_CONV && TILE_W + HKW - 1 == 16 && SWZ == 128 && LINE == 0),
              "halo lines: 3x3-style conv, TILE_W = 17 - KW, 128-byte swizzle");
static_assert(LINE == 0 || (OPEVO_CONV && !HALO && (LINE == 16 || LINE == 32) && TILE_W <= LINE),
              "padded lines: conv, 16 or 32 rows per line of TILE_W pixels");
static_assert(!OPEVO_CONV || ((LINE > 0 ? (TILE_N >= 1 && A_ROWS <= BM_CTA) : A_ROWS == BM_CTA) &&
                              CLUSTER == 1),
              "conv tile must cover BM pixels (padded lines: at most BM), no multicast");

// UMMA instruction descriptor, kind::f16: D=f32, A=B=bf16, both K-major
// (kind::tf32 for X3: A=B=tf32, format code 2).
constexpr u32 AB_FMT = X3 ? 2u : 1u;
constexpr u32 IDESC = (1u << 4) | (AB_FMT << 7) | (AB_FMT << 10) |
                      ((u32)(BN >> 3) << 17) | ((u32)(UMMA_M >> 4) << 24);
static_assert(!X3 || (CG == 1 && CLUSTER == 1 && !OPEVO_CONV && BPU == 1 && OPEVO_ACC == 1 &&
                      OPEVO_TF32X3 > 0 && OPEVO_OUT_F32 && !B_RES),
              "3xTF32: single-CTA GEMM tiles, fp32 output");

// Shared-memory matrix descriptor minus the start address.
constexpr u64 DESC_HI = ((u64)1 << 16)                          // LBO (unused for swizzled K-major)
                      | ((u64)((8 * SWZ) >> 4) << 32)            // SBO: next 8-row group
                      | ((u64)1 << 46)                           // descriptor version (sm_100)
                      | ((u64)LAYOUT << 61);

// TMEM accumulator buffers: two when they fit, so the epilogue of one tile
// overlaps the mainloop of the next (persistent schedule).
// Four when they fit in half of TMEM: a persistent CTA's epilogue then
// trails the MMA by up to three units (the commit -> epilogue -> release
// round trip is long next to a small unit's mainloop).
constexpr int NBUF = (4 * TMEM_USED <= 256) ? 4 : (2 * TMEM_USED <= 512) ? 2 : 1;
// 3xTF32 with A's lo part in TMEM (X3T): the epilogue warps write each landed
// stage's A_lo rows into a TMEM ring after the accumulators (one fp32 per
// column, row = lane) and the A_lo x B MMA reads A from TMEM -- A_lo never
// touches shared memory (its store and its MMA read were a third of the
// stage's shared-memory traffic).  Single-CTA 128-row tiles, 128-byte
// swizzle, when the ring fits next to the accumulators.
constexpr int ALO_COLS = X3 ? BK / 2 : 0;                  // fp32 A elements per row per stage
constexpr bool X3T = X3 && SWZ == 128 && MATOMS == 1 && CG == 1 && BM == 128 && !OPEVO_X3_SMEM_ALO &&
                     NBUF * TMEM_USED + STAGES * ALO_COLS <= 512;
constexpr int ALO_BASE = NBUF * TMEM_USED;                 // first column of the A_lo ring
constexpr int TMEM_NEED = NBUF * TMEM_USED + (X3T ? STAGES * ALO_COLS : 0);
constexpr int TMEM_ALLOC = (TMEM_NEED <= 32) ? 32 : (TMEM_NEED <= 64) ? 64 :
                           (TMEM_NEED <= 128) ? 128 : (TMEM_NEED <= 256) ? 256 : 512;
constexpr int SPLITCL = OPEVO_SPLIT_CLUSTER;   // DSMEM split-K cluster size (0: off)
static_assert(BPU == 1 || (OPEVO_BATCHED && CG == 1 && CLUSTER == 1 && MATOMS == 1 && ACC == 1 &&
                           SPLITCL == 0 && (FUSED_K || KATOMS == 1)),
              "batches per unit: single-CTA 128-row BatchMatMul tiles");
constexpr int CLSZ = CLUSTER * CG * (SPLITCL > 1 ? SPLITCL : 1);   // CTAs per cluster (launch dim x)
// DSMEM reduction buffers (reusing the pipeline smem after the mainloop):
// OWN [BM][RED_LD] fp32, then RECV [SPLITCL-1][BM/SPLITCL][RED_LD] fp32.  Rows
// are padded by 16 B: each epilogue thread stages its own row, and an
// unpadded 512 B row stride would put all 32 lanes on the same banks.
constexpr int RED_LD = BN + 4;
constexpr int RED_ROWS = (SPLITCL > 1) ? BM / SPLITCL : BM;
constexpr int RED_OWN_BYTES = BM * RED_LD * 4;
constexpr int RED_BLOCK_BYTES = RED_ROWS * RED_LD * 4;
constexpr int RED_BYTES = (SPLITCL > 1) ? RED_OWN_BYTES + (SPLITCL - 1) * RED_BLOCK_BYTES : 0;
constexpr int SPLITT = OPEVO_SPLIT_TMA;        // TMA split-K slices (0: off)
// TMA split-K staging in the (then idle) pipeline smem: a slice's fp32 tile
// [BN/32 chunks][BM rows][32] for publishing, or the S-1 peers' tiles for
// reducing
constexpr int SPLITT_BYTES = SPLITT > 1 ? ((SPLITT - 1 > 1 ? SPLITT - 1 : 1) * BM * BN * 4) : 0;
constexpr int PIPE_BYTES0 = (STAGES * STAGE_BYTES > RED_BYTES) ? STAGES * STAGE_BYTES : RED_BYTES;
constexpr int PIPE_BYTES = PIPE_BYTES0 > SPLITT_BYTES ? PIPE_BYTES0 : SPLITT_BYTES;
// Epilogue staging for TMA stores: per epilogue warp two buffers of
// 32 rows x EPI_COLS outputs, laid out in the swizzle the C tensor map uses
// (row bytes 32/64/128 -> SW32/64/128), so the warp's smem writes are
// conflict-free and each chunk leaves as one cp.async.bulk.tensor store.
constexpr int OUT_BYTES = OPEVO_OUT_F32 ? 4 : 2;
constexpr int EPI_ROW_BYTES = STORE_COLS * OUT_BYTES;     // 32, 64 or 128
constexpr int EPI_BUF = 32 * EPI_ROW_BYTES;               // one chunk of one warp
constexpr int EPI_OFF = (PIPE_BYTES + 1023) / 1024 * 1024;
constexpr int EPI_BYTES = 4 * 2 * EPI_BUF;
constexpr int BAR_OFF = EPI_OFF + EPI_BYTES;
// resident weight panel (B_RES): [K/64 atoms][BN rows][128 B], after a
// 1 KB barrier block; its size (BN x K) is a launch-time quantity
constexpr int BRES_OFF = BAR_OFF + 1024;
static_assert(!B_RES || (OPEVO_CONV && SWZ == 128 && CG == 1 && SPLITCL == 0),
              "resident weights: conv, 128-byte swizzle");
static_assert(SPLITT == 0 || ((SPLITT == 2 || SPLITT == 4) && SPLITCL == 0 && CG == 1 && CLUSTER == 1 &&
                           BM == 128 && ACC == 1 && !OPEVO_BATCHED && !OPEVO_CONV && BN % 32 == 0 &&
                           OPEVO_BPU == 1 && !OPEVO_OUT_F32),
              "TMA split-K: S in {2,4}, single-CTA 128-row bf16 GEMM tiles");
static_assert(SPLITCL == 0 || ((SPLITCL == 2 || SPLITCL == 4 || SPLITCL == 8) && CG == 1 && CLUSTER == 1 && !LINES &&
                           MATOMS == 1 && BM % (SPLITCL * 8) == 0),
              "DSMEM split-K: S in {2,4,8}, single-CTA 128-row tiles");

struct __align__(64) TmaDesc { u64 raw[16]; };

// Work decomposition.  A *unit* is what one cluster computes at a time: one
// output tile (CLSZ == 1), CLUSTER column tiles sharing the multicast A tile,
// or one 256-row pair tile (CG == 2); for split-K, one K slice of it.  CTAs
// loop over units (persistent when gridDim < units).
struct Sched {
    int row_tiles;     // tiles along rows (pair tiles for CG == 2)
    int col_groups;    // column tiles / CLUSTER
    int batches;
    int split;         // K slices of every tile (split-K knob)
    int head_tiles;    // tiles computed with `split` slices ...
    int tail_split;    // ... the rest (the last partial wave) with split*tail_split
    int units;         // head_tiles*split + (tiles-head_tiles)*split*tail_split
};

// Conv geometry (unused by the GEMM instances).
struct ConvGeom {
    int cin, ho, wo, kw, pad;
    int taps_cchunks;      // (Cin / BK): K blocks per filter tap (Cin padded to 16)
    int stride;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ u32 smem_u32(const void* p) {
    return (u32)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                 "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1; }"
                 :: "r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ u64 global_ns() {
    u64 t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void mbar_arrive(u32 bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory");
}

// Arrive on a peer CTA's mbarrier (shared::cluster address).  Used only to
// hand a drained TMEM buffer back to the pair leader: the TMEM reads are
// ordered by tcgen05.wait::ld + tcgen05.fence::before_thread_sync, so the
// arrive needs no cluster-scope release (which costs a full memory barrier,
// ~0.5 us, on every epilogue).
__device__ __forceinline__ void mbar_arrive_cluster(u32 cluster_bar) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];"
                 :: "r"(cluster_bar) : "memory");
}

// Parity wait with a watchdog: a configuration that deadlocks traps after
// ~4 s instead of hanging the device (the evaluator scores it 0).
__device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
    u32 done;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                 "selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    if (done) return;
#ifdef OPEVO_NO_WATCHDOG      // debug: plain spin
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                     "selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
#else
    const u64 t0 = global_ns();
    while (true) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                     "selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
        if (done) return;
        if (global_ns() - t0 > 4000000000ull) asm volatile("trap;");
    }
#endif
}

__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ u32 sm_id() {
    u32 r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

#if OPEVO_TRACE == 1
#define TRACE(slot) do { trace[(slot)] = global_ns(); } while (0)
#else
#define TRACE(slot) do { } while (0)
#endif
// OPEVO_TRACE == 2: per-unit handshake stamps of the first five units instead
// (slot 1 + 3u: MMA warp issued unit u's tfull commit; 2 + 3u: epilogue saw
// it; 3 + 3u: epilogue finished unit u) -- tools/trace_units.py
#if OPEVO_TRACE == 2
#define UTRACE(slot) do { trace[(slot)] = global_ns(); } while (0)
#else
#define UTRACE(slot) do { } while (0)
#endif
#if OPEVO_TRACE == 3
#define UTRACE3(slot) do { trace[(slot)] = global_ns(); } while (0)
#else
#define UTRACE3(slot) do { } while (0)
#endif

__device__ __forceinline__ void tma_prefetch(const TmaDesc* d) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(d) : "memory");
}

__device__ __forceinline__ void tma_load_2d(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
                 "[%0], [%1, {%3, %4}], [%2]; }"
                 :: "r"(dst), "l"(d), "r"(bar), "r"(c0), "r"(c1) : "memory");
}

__device__ __forceinline__ void tma_load_3d(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1, int c2) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                 "[%0], [%1, {%3, %4, %5}], [%2]; }"
                 :: "r"(dst), "l"(d), "r"(bar), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

__device__ __forceinline__ void tma_load_4d(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
                 "[%0], [%1, {%3, %4, %5, %6}], [%2]; }"
                 :: "r"(dst), "l"(d), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

__device__ __forceinline__ void tma_load_2d_mc(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1,
                                               u16 mask) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5; }"
                 :: "r"(dst), "l"(d), "r"(bar), "r"(c0), "r"(c1), "h"(mask) : "memory");
}

__device__ __forceinline__ void tma_load_3d_mc(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1,
                                               int c2, u16 mask) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6; }"
                 :: "r"(dst), "l"(d), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "h"(mask) : "memory");
}

// TMA stores (smem -> global) of one epilogue chunk, bulk-group completion
__device__ __forceinline__ void tma_store_2d(const TmaDesc* d, u32 src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 :: "l"(d), "r"(src), "r"(c0), "r"(c1) : "memory");
}

__device__ __forceinline__ void tma_store_3d(const TmaDesc* d, u32 src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                 :: "l"(d), "r"(src), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

__device__ __forceinline__ void tma_store_4d(const TmaDesc* d, u32 src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
                 :: "l"(d), "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}

__device__ __forceinline__ void fence_async_smem() {   // generic-proxy smem writes -> async proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void st_shared_v4(u32 addr, u32 a, u32 b, u32 c, u32 d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__device__ __forceinline__ u32 cluster_rank() {
    u32 r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}

// Issued by a converged warp: one elected lane executes the MMA, so every
// operand stays in uniform registers (no per-MMA R2UR/ELECT loop).
__device__ __forceinline__ void umma_bf16(u32 tmem_d, u64 adesc, u64 bdesc, u32 accumulate) {
    asm volatile("{ .reg .pred e, p; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; "
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                 :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

// One 3xTF32 K step (K8 of fp32 = one 32-byte step): D += A.B_lo + A.B +
// A_lo.B.  The first two share A: the first MMA fills the tensor core's A
// collector buffer and the second reads A from it (lastuse), saving one A
// read from shared memory per step.  kind::tf32 reads the top 19 bits of each fp32
// container (truncation: hi = x & ~0x1fff); the epilogue warps wrote the
// exact remainders lo = x - hi at +LO_OFF, so the
// three products are hi*lo, lo*hi and hi*hi and only lo*lo (~2^-22
// relative) and the tf32 truncation of the lo parts are lost.
// The same three MMAs with A_lo read from TMEM (column address alo_t).
__device__ __forceinline__ void umma_x3t(u32 d, u64 a, u64 b, u32 alo_t, u64 blo, u32 accumulate) {
    asm volatile("{ .reg .pred e, p, t; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %5, 0; "
                 "setp.eq.b32 t, 0, 0; "
                 "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::fill [%0], %1, %4, %6, p; "
                 "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::lastuse [%0], %1, %2, %6, t; "
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%3], %2, %6, t; }"
                 :: "r"(d), "l"(a), "l"(b), "r"(alo_t), "l"(blo), "r"(accumulate), "r"(IDESC));
}

__device__ __forceinline__ void umma_x3(u32 d, u64 a, u64 b, u64 alo, u64 blo, u32 accumulate) {
    asm volatile("{ .reg .pred e, p, t; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %5, 0; "
                 "setp.eq.b32 t, 0, 0; "
                 "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::fill [%0], %1, %4, %6, p; "
                 "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::lastuse [%0], %1, %2, %6, t; "
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %3, %2, %6, t; }"
                 :: "r"(d), "l"(a), "l"(b), "l"(alo), "l"(blo), "r"(accumulate), "r"(IDESC));
}

// All K16 steps of one swizzle atom (NK = ATOM_K / 16 MMAs into one
// accumulator) in one asm block under one elect: the descriptors of steps
// 1.. are the first ones plus 2 * step (32 bytes) in the start-address
// field, computed next to the MMAs, so the issuing warp spends a handful of
// instructions per MMA instead of rebuilding and broadcasting descriptors.
#define OPEVO_UMMA_ATOM(CGS)                                                                          \
    template <int NK>                                                                                \
    __device__ __forceinline__ void umma##CGS##_atom(u32 d, u64 a, u64 b, u32 acc_first);             \
    template <>                                                                                      \
    __device__ __forceinline__ void umma##CGS##_atom<1>(u32 d, u64 a, u64 b, u32 acc_first) {         \
        asm volatile("{ .reg .pred e, p; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; "          \
                     "@e tcgen05.mma.cta_group::" #CGS ".kind::f16 [%0], %1, %2, %3, p; }"            \
                     :: "r"(d), "l"(a), "l"(b), "r"(IDESC), "r"(acc_first));                          \
    }                                                                                                \
    template <>                                                                                      \
    __device__ __forceinline__ void umma##CGS##_atom<2>(u32 d, u64 a, u64 b, u32 acc_first) {         \
        asm volatile("{ .reg .pred e, p, t; .reg .b64 a1, b1; elect.sync _|e, 0xffffffff; "           \
                     "setp.ne.b32 p, %4, 0; setp.eq.b32 t, 0, 0; add.s64 a1, %1, 2; add.s64 b1, %2, 2; " \
                     "@e tcgen05.mma.cta_group::" #CGS ".kind::f16 [%0], %1, %2, %3, p; "             \
                     "@e tcgen05.mma.cta_group::" #CGS ".kind::f16 [%0], a1, b1, %3, t; }"            \
                     :: "r"(d), "l"(a), "l"(b), "r"(IDESC), "r"(acc_first));                          \
    }                                                                                                \
    template <>                                                                                      \
    __device__ __forceinline__ void umma##CGS##_atom<4>(u32 d, u64 a, u64 b, u32 acc_first) {         \
        asm volatile("{ .reg .pred e, p, t; .reg .b64 a1, b1, a2, b2, a3, b3; elect.sync _|e, 0xffffffff; " \
                     "setp.ne.b32 p, %4, 0; setp.eq.b32 t, 0, 0; "                                    \
                     "add.s64 a1, %1, 2; add.s64 b1, %2, 2; add.s64 a2, %1, 4; add.s64 b2, %2, 4; "  \
                     "add.s64 a3, %1, 6; add.s64 b3, %2, 6; "                                         \
                     "@e tcgen05.mma.cta_group::" #CGS ".kind::f16 [%0], %1, %2, %3, p; "             \
                     "@e tcgen05.mma.cta_group::" #CGS ".kind::f16 [%0], a1, b1, %3, t; "             \
                     "@e tcgen05.mma.cta_group::" #CGS ".kind::f16 [%0], a2, b2, %3, t; "             \
                     "@e tcgen05.mma.cta_group::" #CGS ".kind::f16 [%0], a3, b3, %3, t; }"            \
                     :: "r"(d), "l"(a), "l"(b), "r"(IDESC), "r"(acc_first));                          \
    }
OPEVO_UMMA_ATOM(1)
OPEVO_UMMA_ATOM(2)
#undef OPEVO_UMMA_ATOM

__device__ __forceinline__ void umma_commit(u32 bar) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }"
                 :: "r"(bar) : "memory");
}

// CTA-pair variants (cta_group::2)
__device__ __forceinline__ void umma2_bf16(u32 tmem_d, u64 adesc, u64 bdesc, u32 accumulate) {
    asm volatile("{ .reg .pred e, p; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; "
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p; }"
                 :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void umma2_commit_mc(u32 bar, u16 mask) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster"
                 ".multicast::cluster.b64 [%0], %1; }" :: "r"(bar), "h"(mask) : "memory");
}

// TMA load whose completion is credited to the pair leader's mbarrier
// (`bar` is a shared::cluster address from mapa).
__device__ __forceinline__ void tma2_load_2d(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e cp.async.bulk.tensor.2d.cta_group::2"
                 ".shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2]; }"
                 :: "r"(dst), "l"(d), "r"(bar), "r"(c0), "r"(c1) : "memory");
}

__device__ __forceinline__ void tma2_load_3d(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1, int c2) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e cp.async.bulk.tensor.3d.cta_group::2"
                 ".shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2]; }"
                 :: "r"(dst), "l"(d), "r"(bar), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

__device__ __forceinline__ void tma2_load_4d(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1, int c2,
                                             int c3) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e cp.async.bulk.tensor.4d.cta_group::2"
                 ".shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2]; }"
                 :: "r"(dst), "l"(d), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

__device__ __forceinline__ u32 mapa_cta(u32 addr, u32 rank) {
    u32 r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

// Conv operand loads: plain, or (CTA pair) credited to the leader's barrier.
__device__ __forceinline__ void conv_load_a(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1, int c2,
                                            int c3) {
    if (CG == 2) tma2_load_4d(dst, d, bar, c0, c1, c2, c3);
    else         tma_load_4d(dst, d, bar, c0, c1, c2, c3);
}

__device__ __forceinline__ void conv_load_b(u32 dst, const TmaDesc* d, u32 bar, int c0, int c1) {
    if (CG == 2) tma2_load_2d(dst, d, bar, c0, c1);
    else         tma_load_2d(dst, d, bar, c0, c1);
}

// Halo lines: all KW weight tiles of one filter row (and every 64-channel atom
// of the K block) in ONE box {64, BN_LOAD, KATOMS, KW} of the weight view
// {64, Cout, Cin/64, KH*KW}; it lands [tap][atom][row][128 B], the layout the
// MMA descriptors walk (tap stride B_SUB).
__device__ __forceinline__ void conv_load_b_row(u32 dst, const TmaDesc* d, u32 bar, int row0, int atom0,
                                                int tap0) {
    if (CG == 2) tma2_load_4d(dst, d, bar, 0, row0, atom0, tap0);
    else         tma_load_4d(dst, d, bar, 0, row0, atom0, tap0);
}

__device__ __forceinline__ void umma_commit_mc(u32 bar, u16 mask) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; "
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster"
                 ".multicast::cluster.b64 [%0], %1; }" :: "r"(bar), "h"(mask) : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void epi_bar() {   // the four epilogue warps only
    asm volatile("bar.sync 1, 128;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void tmem_load(u32 taddr, u32 (&v)[N]);

template <>
__device__ __forceinline__ void tmem_load<32>(u32 taddr, u32 (&v)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                   "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                   "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                   "=r"(v[30]), "=r"(v[31])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <>
__device__ __forceinline__ void tmem_load<64>(u32 taddr, u32 (&v)[64]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <>
__device__ __forceinline__ void tmem_load<16>(u32 taddr, u32 (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                   "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ u32 pack_bf16(float lo, float hi) {
    u32 r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ void st_v4(void* p, u32 a, u32 b, u32 c, u32 d) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" :: "l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__device__ __forceinline__ u32 atom_add_release_gpu(u32* p, u32 v) {
    u32 old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void fence_acq_rel_gpu() {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__device__ __forceinline__ float4 ld_cg_f4(const float* p) {
    float4 r;
    asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}

// Sum the ACC interleaved accumulators of one row segment (fixed order).
template <int N = EPI_COLS>
__device__ __forceinline__ void gather_acc(u32 taddr, float (&out)[N]) {
    u32 v[N];
    tmem_load<N>(taddr, v);
#pragma unroll
    for (int j = 0; j < N; ++j) out[j] = __uint_as_float(v[j]);
#pragma unroll
    for (int a = 1; a < ACC; ++a) {
        tmem_load<N>(taddr + a * MATOMS * BN, v);
#pragma unroll
        for (int j = 0; j < N; ++j) out[j] += __uint_as_float(v[j]);
    }
}

// Stage one thread's row (EPI_COLS outputs) of a 32-row epilogue chunk in the
// TMA swizzle of the C map: 16-byte unit j of row r lands at unit
// j ^ ((r * EPI_ROW_BYTES / 128) mod units), i.e. SW128/SW64/SW32 for 128/64/32-byte rows.
__device__ __forceinline__ void stage_row(u32 buf, int r, const float (&acc)[STORE_COLS]) {
    constexpr int UNITS = EPI_ROW_BYTES / 16;
    const u32 row = buf + (u32)(r * EPI_ROW_BYTES);
    const int x = ((r * EPI_ROW_BYTES) >> 7) & (UNITS - 1);
#pragma unroll
    for (int j = 0; j < UNITS; ++j) {
        const u32 dst = row + (u32)((j ^ x) << 4);
#if OPEVO_OUT_F32
        st_shared_v4(dst, __float_as_uint(acc[4 * j]), __float_as_uint(acc[4 * j + 1]),
                     __float_as_uint(acc[4 * j + 2]), __float_as_uint(acc[4 * j + 3]));
#else
        st_shared_v4(dst, pack_bf16(acc[8 * j], acc[8 * j + 1]), pack_bf16(acc[8 * j + 2], acc[8 * j + 3]),
                     pack_bf16(acc[8 * j + 4], acc[8 * j + 5]), pack_bf16(acc[8 * j + 6], acc[8 * j + 7]));
#endif
    }
}

// fp32 row of a 32-column chunk (128 bytes) in the SW128 layout of tma_w.
__device__ __forceinline__ void stage_row_f32(u32 buf, int r, const float* acc) {
    const u32 row = buf + (u32)(r * 128);
#pragma unroll
    for (int j = 0; j < 8; ++j)
        st_shared_v4(row + (u32)((j ^ (r & 7)) << 4), __float_as_uint(acc[4 * j]), __float_as_uint(acc[4 * j + 1]),
                     __float_as_uint(acc[4 * j + 2]), __float_as_uint(acc[4 * j + 3]));
}

__device__ __forceinline__ void add_row_f32(u32 buf, int r, float* acc) {
    const u32 row = buf + (u32)(r * 128);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(row + (u32)((j ^ (r & 7)) << 4)));
        acc[4 * j] += v.x; acc[4 * j + 1] += v.y; acc[4 * j + 2] += v.z; acc[4 * j + 3] += v.w;
    }
}

__device__ __forceinline__ u32 ld_acquire_gpu(const u32* p) {
    u32 v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Write EPI_COLS fp32 accumulator values (one row segment) as the output type.
__device__ __forceinline__ void store_row(void* c_out, u64 off, const float* acc) {
#if OPEVO_OUT_F32
    float* dst = reinterpret_cast<float*>(c_out) + off;
#pragma unroll
    for (int j = 0; j < EPI_COLS; j += 4)
        st_v4(dst + j, __float_as_uint(acc[j]), __float_as_uint(acc[j + 1]),
              __float_as_uint(acc[j + 2]), __float_as_uint(acc[j + 3]));
#else
    u16* dst = reinterpret_cast<u16*>(c_out) + off;
#pragma unroll
    for (int j = 0; j < EPI_COLS; j += 8)
        st_v4(dst + j, pack_bf16(acc[j], acc[j + 1]), pack_bf16(acc[j + 2], acc[j + 3]),
              pack_bf16(acc[j + 4], acc[j + 5]), pack_bf16(acc[j + 6], acc[j + 7]));
#endif
}

}  // namespace opevo

using namespace opevo;

extern "C" __global__ void __launch_bounds__(NUM_THREADS, 2)   // 2: keep <= 168 regs so two CTAs can co-reside
opevo_gemm(const __grid_constant__ TmaDesc tma_a,
           const __grid_constant__ TmaDesc tma_b,
           const __grid_constant__ TmaDesc tma_c,   // C, box = 32 rows x EPI_COLS (TMA-store epilogue)
           const __grid_constant__ TmaDesc tma_w,   // split-K partials {cols, rows, split} fp32, box 32 x 32
           void* __restrict__ c_out,
           float* __restrict__ ws,            // split-K partials [split][batch*rows][cols]
           u32* __restrict__ counters,        // per-tile arrival counters (self-resetting)
           int rows, int cols, int depth,      // depth = K (per batch)
           const Sched sched,
           const ConvGeom geom)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<u64>(smem_raw) + SMEM_ALIGN - 1) & ~(u64)(SMEM_ALIGN - 1));
    u64* full_bar = reinterpret_cast<u64*>(smem + BAR_OFF);
    u64* empty_bar = full_bar + STAGES;
    u64* tfull_bar = empty_bar + STAGES;      // MMA -> epilogue, per TMEM buffer
    u64* tempty_bar = tfull_bar + NBUF;       // epilogue -> MMA, per TMEM buffer
    u64* red_bar = tempty_bar + NBUF;         // DSMEM split-K: peers' partial rows landed
    u64* bres_bar = red_bar + 1;              // weight panel landed (B_RES)
    u64* part_bar = bres_bar + 1;             // TMA split-K: peers' partials landed, per epilogue warp
    u64* lo_bar = part_bar + 4;               // X3: stage split into hi/lo (epilogue warps -> MMA)
    u32* tmem_slot = reinterpret_cast<u32*>(lo_bar + (X3 ? STAGES : 0));
    u32* last_flag = tmem_slot + 1;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const u32 crank = (CLSZ > 1) ? cluster_rank() : 0u;
    const u32 prank = (CG == 2) ? crank : 0u;                 // rank in the CTA pair
    const u32 mrank = (CLUSTER > 1) ? crank : 0u;            // rank in a multicast cluster
    const int cl_id = (int)(blockIdx.x / CLSZ);
    const int cl_count = (int)(gridDim.x / CLSZ);
    // work items: one per cluster at a time; a DSMEM split-K cluster's CTAs
    // each own one K slice (unit) of the same tile
    const int u_first = (SPLITCL > 1) ? (int)blockIdx.x : cl_id;
    const int u_step = (SPLITCL > 1) ? (int)gridDim.x : cl_count;
    const int head_items = sched.head_tiles * sched.split;
#if OPEVO_TRACE
    u64* trace = reinterpret_cast<u64*>(ws) + 16ull * blockIdx.x;
    if (threadIdx.x == 0) { trace[0] = sm_id(); TRACE(1); }
#endif
    if (threadIdx.x == 0) pdl_launch_dependents();
    if (OPEVO_ABLATE == 1) return;
    if (OPEVO_ABLATE == 5) asm volatile("trap;");
    (void)mrank;
    (void)geom;

    // unit -> (batch, row tile, column group, K slice); column groups vary
    // fastest so concurrently running clusters share A row panels in L2.
    // Tiles past head_tiles (the last, partial wave of a persistent grid)
    // are cut into tail_split times more K slices so the wave fills up.
    struct Unit { int batch, row_tile, col_tile, kz, split, k0, num_kb; };
    auto decode = [&](int u) -> Unit {
        Unit t;
        if (u < head_items) {
            t.split = sched.split;
            t.kz = u % t.split;
            u /= t.split;
        } else {
            const int v = u - head_items;
            t.split = sched.split * sched.tail_split;
            t.kz = v % t.split;
            u = sched.head_tiles + v / t.split;
        }
        const int klen = depth / t.split;
        t.k0 = t.kz * klen;
        t.num_kb = (OPEVO_ABLATE == 2 || OPEVO_ABLATE == 7) ? 0 : klen / BK;
        const int colg = u % sched.col_groups;
        u /= sched.col_groups;
        t.row_tile = u % sched.row_tiles;
        t.batch = u / sched.row_tiles;
        t.col_tile = colg * CLUSTER + (int)mrank;
        return t;
    };

    // Incremental walk over this CTA's units u_first, u_first + u_step, ...:
    // the mixed-radix digits (K slice, column group, row tile, batch) of the
    // step are computed once, so advancing costs adds and compares instead
    // of decode()'s divisions on every unit in three warps (decode remains
    // for the K-split tail of grid mode 2).
    struct UnitWalk { int u, kz, colg, row, batch; };
    const int klen0 = depth / sched.split;
    const int num_kb0 = (OPEVO_ABLATE == 2 || OPEVO_ABLATE == 7) ? 0 : klen0 / BK;
    auto digits = [&](int q) -> UnitWalk {
        UnitWalk w;
        w.u = q;
        w.kz = q % sched.split; q /= sched.split;
        w.colg = q % sched.col_groups; q /= sched.col_groups;
        w.row = q % sched.row_tiles;
        w.batch = q / sched.row_tiles;
        return w;
    };
    const UnitWalk step = digits(u_step);
    auto walk_next = [&](UnitWalk& w) {
        w.u += u_step;
        w.kz += step.kz;
        int c = w.kz >= sched.split;
        if (c) w.kz -= sched.split;
        w.colg += step.colg + c;
        c = w.colg >= sched.col_groups;
        if (c) w.colg -= sched.col_groups;
        w.row += step.row + c;
        c = w.row >= sched.row_tiles;
        if (c) w.row -= sched.row_tiles;
        w.batch += step.batch + c;
    };
    auto unit_of = [&](const UnitWalk& w) -> Unit {
        if (w.u >= head_items) return decode(w.u);
        Unit t;
        t.split = sched.split;
        t.kz = w.kz;
        t.k0 = w.kz * klen0;
        t.num_kb = num_kb0;
        t.row_tile = w.row;
        t.batch = w.batch;
        t.col_tile = w.colg * CLUSTER + (int)mrank;
        return t;
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        tma_prefetch(&tma_c);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(full_bar + s), 1);
            // with multicast every CTA of the cluster must release a slot
            // before any of them overwrites it
            mbar_init(smem_u32(empty_bar + s), CG == 2 ? 1 : CLUSTER);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(smem_u32(tfull_bar + b), 1);
            // one arrival per epilogue warp; a pair leader's MMAs also write
            // the peer's TMEM, so it waits for both CTAs' epilogues
            mbar_init(smem_u32(tempty_bar + b), 4 * CG);
        }
        if (SPLITCL > 1) {
            // one phase per launch: expect the (SPLITCL-1) row blocks the peers push
            mbar_init(smem_u32(red_bar), 1);
        }
        if (B_RES) mbar_init(smem_u32(bres_bar), 1);
        if (SPLITT > 1)
            for (int q = 0; q < 4; ++q) mbar_init(smem_u32(part_bar + q), 1);
        if (X3)
            for (int q = 0; q < STAGES; ++q) mbar_init(smem_u32(lo_bar + q), 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (SPLITCL > 1)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                         :: "r"(smem_u32(red_bar)), "r"((u32)((SPLITCL - 1) * RED_BLOCK_BYTES)) : "memory");
    }
    __syncwarp();
    // Publish the barrier inits cluster-wide now (every warp arrives before
    // its own setup work); each role waits at the end of setup.
    if (CLSZ > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    if (warp == 1) {
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                         :: "r"(smem_u32(tmem_slot)), "r"(TMEM_ALLOC) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                         :: "r"(smem_u32(tmem_slot)), "r"(TMEM_ALLOC) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    // The producer only needs its own warp's barrier inits (and, in a
    // cluster, the peers'): it arrives on named barrier 2 without waiting,
    // so its first TMA does not wait for the TMEM allocation; the MMA and
    // epilogue warps wait for both the inits and the allocation.
    tc_fence_before();
    if (warp == 0) asm volatile("bar.arrive 2, %0;" :: "n"(NUM_THREADS) : "memory");
    else           asm volatile("bar.sync 2, %0;" :: "n"(NUM_THREADS) : "memory");
    if (CLSZ > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const u32 tmem_base = (warp == 0) ? 0u : __shfl_sync(0xffffffffu, *tmem_slot, 0);   // warp-uniform
    if (threadIdx.x == 0) TRACE(2);

    if (warp == 0) {
        // ---------------------------------------------------- TMA producer
        // (whole warp iterates; the tma_* / expect_tx helpers elect one lane)
        int s = 0;
        u32 ph = 0;
        int issued = 0;                 // k-blocks issued; the first STAGES slots start free
        bool first = true;
        // everything up to the first global read happens before the PDL wait
        UnitWalk w = digits(u_first);
        const Unit t_first = unit_of(w);
        pdl_wait();                     // operands may be the previous launch's output
        if (lane == 0) TRACE(9);
#if OPEVO_CONV
        if (B_RES && w.u < sched.units) {
            // the whole weight panel of this CTA's column tile, once: one box
            // {64, BN, K/64} of the atom view lands it atom-major
            // (halo lines: the kernel's K loop runs over filter rows only,
            // depth = KH * Cin, while the panel holds all KH * KW taps)
            const u32 bytes = (u32)BN * (u32)depth * (HALO ? (u32)HKW : 1u) * 2u;
            mbar_expect_tx(smem_u32(bres_bar), bytes);
            tma_load_3d(smem_u32(smem + BRES_OFF), &tma_b, smem_u32(bres_bar), 0, t_first.col_tile * BN, 0);
        }
#endif
        for (; w.u < sched.units; walk_next(w)) {
            const Unit t = (w.u == u_first) ? t_first : unit_of(w);
            const int k0 = t.k0;
            const int num_kb = t.num_kb;
            const int col0 = t.col_tile * BN;
#if OPEVO_CONV
            const int w_tiles = geom.wo / TILE_W, h_tiles = geom.ho / TILE_H;
            const int w0 = (t.row_tile % w_tiles) * TILE_W;
            const int h0 = ((t.row_tile / w_tiles) % h_tiles) * TILE_H;
            const int n0 = (t.row_tile / (w_tiles * h_tiles)) * PAIR_TN + (int)prank * TILE_N;
            const int b_row0 = col0 + (int)prank * BN_LOAD;         // first B row here
#else
            const int row0 = t.row_tile * BM + (int)prank * BM_CTA;   // first A row here
            const int b_row0 = col0 + (int)prank * BN_LOAD;         // first B row here
#endif
            for (int kb = 0; kb < num_kb; ++kb) {
                if (issued >= STAGES) mbar_wait(smem_u32(empty_bar + s), ph ^ 1);
                ++issued;
                if (first && lane == 0) TRACE(10);
                const u32 fb = (CG == 2) ? mapa_cta(smem_u32(full_bar + s), 0) : smem_u32(full_bar + s);
                if (OPEVO_ABLATE == 3) {
                    if (lane == 0) mbar_arrive(fb);
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                    continue;
                }
                if (prank == 0) mbar_expect_tx(smem_u32(full_bar + s), TX_STAGE);
                if (first && lane == 0) TRACE(11);
                const u32 a_dst = smem_u32(smem + s * STAGE_BYTES);
                const u32 b_dst = a_dst + A_TILE;
                const int kk = k0 + kb * BK;
#if OPEVO_CONV
                const int kblk = kk / BK;                    // global K block
                const int tap = kblk / geom.taps_cchunks;    // halo lines: the filter row
                const int cbase = (kblk - tap * geom.taps_cchunks) * BK;
                if (HALO) {
                    // one box of 16-pixel lines (the KW taps of filter row `tap`
                    // read it at row offsets 0..KW-1) plus, streamed, the KW
                    // weight tiles of that filter row
                    const int di = tap - geom.pad;
#pragma unroll
                    for (int ka = 0; ka < KATOMS; ++ka)
                        conv_load_a(a_dst + ka * (BM_CTA * SWZ), &tma_a, fb, cbase + ka * ATOM_K,
                                    w0 - geom.pad, h0 + di, n0);
                    if (!B_RES) {
                        if (OPEVO_WBOX) {
                            conv_load_b_row(b_dst, &tma_b, fb, b_row0, cbase / ATOM_K, tap * HKW);
                        } else {    // experiment: one 2-D box per (tap, atom)
#pragma unroll
                            for (int ka = 0; ka < KATOMS; ++ka)
#pragma unroll
                                for (int dj = 0; dj < HKW; ++dj)
                                    conv_load_b(b_dst + dj * B_SUB + ka * (BN_LOAD * SWZ), &tma_b, fb,
                                                (tap * HKW + dj) * geom.cin + cbase + ka * ATOM_K, b_row0);
                        }
                    }
                } else {
                // input pixel of output (h0, w0) under tap (di, dj): the map
                // traverses W and H with element stride S
                const int di = tap / geom.kw - geom.pad, dj = tap % geom.kw - geom.pad;
#pragma unroll
                for (int ka = 0; ka < KATOMS; ++ka) {
                    conv_load_a(a_dst + ka * (BM_CTA * SWZ), &tma_a, fb, cbase + ka * ATOM_K,
                                w0 * geom.stride + dj, h0 * geom.stride + di, n0);
                    if (!B_RES)
                        conv_load_b(b_dst + ka * (BN_LOAD * SWZ), &tma_b, fb, kk + ka * ATOM_K, b_row0);
                }
                }
#else
                if (FUSED_K) {
                    const int katom = kk / ATOM_K;
#if OPEVO_CTA_GROUP == 2
#if OPEVO_BATCHED
                    tma2_load_4d(a_dst, &tma_a, fb, 0, row0, katom, t.batch);
                    tma2_load_4d(b_dst, &tma_b, fb, 0, b_row0, katom, t.batch);
#else
                    tma2_load_3d(a_dst, &tma_a, fb, 0, row0, katom);
                    tma2_load_3d(b_dst, &tma_b, fb, 0, b_row0, katom);
#endif
#else
#if OPEVO_BATCHED
                    tma_load_4d(a_dst, &tma_a, fb, 0, row0, katom, t.batch * BPU);
                    tma_load_4d(b_dst, &tma_b, fb, 0, b_row0, katom, t.batch * BPU);
#else
                    tma_load_3d(a_dst, &tma_a, fb, 0, row0, katom);
                    tma_load_3d(b_dst, &tma_b, fb, 0, b_row0, katom);
#endif
#endif
                } else
#pragma unroll
                for (int ka = 0; ka < KATOMS; ++ka) {
                    const int kc = kk + ka * ATOM_K;
                    const u32 a_sub = a_dst + ka * (BM_CTA * SWZ);
                    const u32 b_sub = b_dst + ka * (BN_LOAD * SWZ);
#if OPEVO_CTA_GROUP == 2
#if OPEVO_BATCHED
                    tma2_load_3d(a_sub, &tma_a, fb, kc, row0, t.batch);
                    tma2_load_3d(b_sub, &tma_b, fb, kc, b_row0, t.batch);
#else
                    tma2_load_2d(a_sub, &tma_a, fb, kc, row0);
                    tma2_load_2d(b_sub, &tma_b, fb, kc, b_row0);
#endif
#else
#if OPEVO_CLUSTER > 1
                    // this CTA fetches one 1/CLUSTER slice of the shared A tile
                    // and multicasts it into every CTA of the cluster
                    const u32 a_part = a_sub + mrank * (A_SLICE_ROWS * SWZ);
                    const u16 mask = (u16)((1u << CLUSTER) - 1);
#if OPEVO_BATCHED
                    tma_load_3d_mc(a_part, &tma_a, fb, kc, row0 + mrank * A_SLICE_ROWS, t.batch, mask);
#else
                    tma_load_2d_mc(a_part, &tma_a, fb, kc, row0 + mrank * A_SLICE_ROWS, mask);
#endif
#else
#if OPEVO_BATCHED
                    tma_load_3d(a_sub, &tma_a, fb, kc, row0, t.batch * BPU);
#else
                    tma_load_2d(a_sub, &tma_a, fb, kc, row0);
#endif
#endif
#if OPEVO_BATCHED
                    tma_load_3d(b_sub, &tma_b, fb, kc, b_row0, t.batch * BPU);
#else
                    tma_load_2d(b_sub, &tma_b, fb, kc, b_row0);
#endif
#endif
                }
#endif
                if (first && lane == 0) { TRACE(3); first = false; }
                if (++s == STAGES) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (CG == 1 || prank == 0) {
            // ------------------------------------------------ MMA issuer
            // (whole warp iterates; umma_* elect one lane to issue)
            int s = 0, buf = 0, mu = 0;   // mu: units committed (trace)
            (void)mu;
            u32 ph = 0, bph = 0;
            bool first = true;
            // Shared-memory descriptors of stage 0; every other operand
            // descriptor is this plus a compile-time offset (>> 4) in the
            // start-address field, which cannot carry out of its 14 bits
            // (shared offsets < 228 KB), so each MMA costs two 64-bit adds
            // rather than a rebuild from the address.
            const u64 desc_a0 = DESC_HI | (u64)((smem_u32(smem) >> 4) & 0x3FFF);
            const u64 desc_b0 = desc_a0 + (u64)(A_TILE >> 4);
            const u64 desc_bres = DESC_HI | (u64)((smem_u32(smem + BRES_OFF) >> 4) & 0x3FFF);
            if (B_RES) mbar_wait(smem_u32(bres_bar), 0);     // the resident weight panel
            // halo + resident weights: descriptor steps through the panel
            // (atom = (BN x 128 B) >> 4 per 64 channels; C/64 atoms per tap
            // column; (KW - 1) columns skipped when a filter row is done)
            constexpr int bres_atom = (BN * SWZ) >> 4;
            const u64 bres_dj = (HALO && B_RES) ? (u64)(geom.cin / 64) * (u64)bres_atom : 0ull;
            const u64 bres_wrap = (u64)(HKW > 0 ? HKW - 1 : 0) * bres_dj;
            (void)bres_wrap;
            for (UnitWalk w = digits(u_first); w.u < sched.units; walk_next(w)) {
                const Unit tu = unit_of(w);
                const int num_kb = tu.num_kb;
                // the epilogue must have drained this accumulator buffer
                mbar_wait(smem_u32(tempty_bar + buf), bph ^ 1);
                tc_fence_after();
                if (lane == 0 && mu < 5) UTRACE3(1 + 3 * mu);
                const u32 acc_base = tmem_base + (u32)(buf * TMEM_USED);
                u64 bres_kb = desc_bres;       // halo + resident weights: this K block's panel atom
                int bres_cch = 0;              // ... and its channel block within the filter row
                (void)bres_kb;
                (void)bres_cch;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(smem_u32(full_bar + s), ph);
                    if (kb == 0 && lane == 0 && mu < 5) UTRACE3(2 + 3 * mu);
                    if (X3) mbar_wait(smem_u32(lo_bar + s), ph);
                    tc_fence_after();
                    if (first && lane == 0) { TRACE(4); first = false; }
                    if (OPEVO_ABLATE == 4) {
                        if (lane == 0) mbar_arrive(smem_u32(empty_bar + s));
                        if (++s == STAGES) { s = 0; ph ^= 1; }
                        continue;
                    }
                    const u64 sdesc = (u64)((u32)(s * STAGE_BYTES) >> 4);
                    // B: this stage's slot, or the resident panel's atoms of this K block
                    const u64 da = desc_a0 + sdesc;
                    const u64 db = B_RES ? desc_bres + (u64)(((tu.k0 / BK + kb) * KATOMS * (BN * SWZ)) >> 4)
                                         : desc_b0 + sdesc;
                    if (HALO) {
                        // filter row `tap` of this K block: tap dj reads the
                        // halo box dj rows further on.  Resident weights: the
                        // panel atom of (row, channel block, dj, ka) is
                        // row*KW*C/64 + dj*C/64 + chunk*KATOMS + ka, walked
                        // incrementally (bres_kb) -- no division or multiply
                        // by runtime values in the MMA warp's loop, whose
                        // instruction count paces the N = 64 MMAs
#pragma unroll
                        for (int dj = 0; dj < HKW; ++dj) {
#pragma unroll
                            for (int ka = 0; ka < KATOMS; ++ka) {
                                const u64 bdesc = B_RES
                                    ? bres_kb + (u64)dj * bres_dj + (u64)(ka * bres_atom)
                                    : db + (u64)((dj * B_SUB + ka * (BN_LOAD * SWZ)) >> 4);
                                // (tap, atom) steps round-robin over ACC accumulators
                                const int step = dj * KATOMS + ka;
                                const int acc = step % ACC;
#pragma unroll
                                for (int ma = 0; ma < MATOMS; ++ma) {
                                    const u64 adesc = da + (u64)((ka * (BM_CTA * SWZ) + ma * (128 * SWZ) + dj * 128) >> 4);
                                    const u32 accumulate = (kb != 0 || step >= ACC) ? 1u : 0u;
                                    const u32 d = acc_base + (u32)((acc * MATOMS + ma) * BN);
                                    if (CG == 2) umma2_atom<ATOM_K / 16>(d, adesc, bdesc, accumulate);
                                    else         umma1_atom<ATOM_K / 16>(d, adesc, bdesc, accumulate);
                                }
                            }
                        }
                    } else if (X3) {
#pragma unroll
                        for (int ka = 0; ka < KATOMS; ++ka) {
#pragma unroll
                            for (int k16 = 0; k16 < ATOM_K / 16; ++k16) {
                                const u32 koff = k16 * 32;
                                const u64 bdesc = db + (u64)((ka * (BN_LOAD * SWZ) + koff) >> 4);
#pragma unroll
                                for (int ma = 0; ma < MATOMS; ++ma) {
                                    const u64 adesc = da + (u64)((ka * (BM_CTA * SWZ) + ma * (128 * SWZ) + koff) >> 4);
                                    const u32 accumulate = (kb != 0 || ka != 0 || k16 != 0) ? 1u : 0u;
                                    if (X3T)
                                        umma_x3t(acc_base + (u32)(ma * BN), adesc, bdesc,
                                                 tmem_base + (u32)(ALO_BASE + s * ALO_COLS + ka * 32 + k16 * 8),
                                                 bdesc + (u64)(LO_OFF >> 4), accumulate);
                                    else
                                        umma_x3(acc_base + (u32)(ma * BN), adesc, bdesc, adesc + (u64)(LO_OFF >> 4),
                                                bdesc + (u64)(LO_OFF >> 4), accumulate);
                                }
                            }
                        }
                    } else if (MATOMS == 1 && ACC == 1) {
                        // one accumulator per batch of the unit: each swizzle
                        // atom's K16 steps in one asm block
#pragma unroll
                        for (int j = 0; j < BPU; ++j) {
#pragma unroll
                        for (int ka = 0; ka < KATOMS; ++ka) {
                            const u64 adesc = da + (u64)((j * A_SUB + ka * (BM_CTA * SWZ)) >> 4);
                            const u64 bdesc = db + (u64)((j * B_SUB + ka * (BN_LOAD * SWZ)) >> 4);
                            const u32 accumulate = (kb != 0 || ka != 0) ? 1u : 0u;
                            const u32 d = acc_base + (u32)(j * BN);
                            if (CG == 2) umma2_atom<ATOM_K / 16>(d, adesc, bdesc, accumulate);
                            else         umma1_atom<ATOM_K / 16>(d, adesc, bdesc, accumulate);
                        }
                        }
                    } else {
#pragma unroll
                    for (int ka = 0; ka < KATOMS; ++ka) {
#pragma unroll
                        for (int k16 = 0; k16 < ATOM_K / 16; ++k16) {
                            const u32 koff = k16 * 32;
                            const u64 bdesc = db + (u64)((ka * (BN_LOAD * SWZ) + koff) >> 4);
#pragma unroll
                            for (int ma = 0; ma < MATOMS; ++ma) {
                                const u64 adesc = da + (u64)((ka * (BM_CTA * SWZ) + ma * (128 * SWZ) + koff) >> 4);
                                const int step = ka * (ATOM_K / 16) + k16;   // k16 step in stage
                                const int acc = step % ACC;                  // compile-time
                                const u32 d = acc_base + (u32)((acc * MATOMS + ma) * BN);
                                const u32 accumulate = (kb != 0 || step >= ACC) ? 1u : 0u;
                                if (CG == 2) umma2_bf16(d, adesc, bdesc, accumulate);
                                else         umma_bf16(d, adesc, bdesc, accumulate);
                            }
                        }
                    }
                    }
#if OPEVO_CTA_GROUP == 2
                    // both CTAs staged this slot: release it in both
                    umma2_commit_mc(smem_u32(empty_bar + s), (u16)3);
#elif OPEVO_CLUSTER > 1
                    // the slot is refilled by multicasts from every cluster CTA:
                    // release it in all of them once our MMAs have consumed it
                    umma_commit_mc(smem_u32(empty_bar + s), (u16)((1u << CLUSTER) - 1));
#else
                    umma_commit(smem_u32(empty_bar + s));
#endif
                    if (HALO && B_RES) {
                        bres_kb += (u64)(KATOMS * bres_atom);
                        if (++bres_cch == geom.taps_cchunks) { bres_cch = 0; bres_kb += bres_wrap; }
                    }
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
                if (CG == 2) umma2_commit_mc(smem_u32(tfull_bar + buf), (u16)3);   // both halves
                else         umma_commit(smem_u32(tfull_bar + buf));
                if (lane == 0 && mu < 5) UTRACE(1 + 3 * mu);
                if (lane == 0 && mu < 5) UTRACE3(3 + 3 * mu);
                ++mu;
                if (++buf == NBUF) { buf = 0; bph ^= 1; }
            }
            if (lane == 0) TRACE(5);
        }
    } else {
        // ---------------------------------------------------- epilogue
        const int quarter = warp & 3;              // TMEM lane quarter of this warp
        const int epi_tid = threadIdx.x - 64;
        const u64 plane = (u64)rows * (u64)cols;   // one batch (or one split slice)
        const u64 slice = (u64)sched.batches * plane;
        // TMEM release target: the pair leader's barrier for CG == 2
        const u32 tempty_leader0 = (CG == 2) ? mapa_cta(smem_u32(tempty_bar), 0) : 0u;
        int buf = 0;
        u32 bph = 0;
        bool first = true;
        const u32 epi_stage = smem_u32(smem + EPI_OFF) + (u32)(quarter * 2 * EPI_BUF);
        int nchunk = 0;                            // TMA-store chunks issued by this warp
        int eu = 0;                                // units drained (trace)
        (void)eu;
#if OPEVO_TF32X3
        int xs = 0;                                // ring slot / phase of the hi/lo split
        u32 xph = 0;
#endif
        for (UnitWalk w = digits(u_first); w.u < sched.units; walk_next(w)) {
            const Unit t = unit_of(w);
            const int col0 = t.col_tile * BN;
#if OPEVO_TF32X3
            // Split every landed stage of this unit: lo = x - hi (exact in
            // fp32) at +LO_OFF, where hi = x with the low 13 mantissa bits
            // cleared -- exactly what kind::tf32 reads from the landed x, so
            // x itself serves as hi (writing hi back in place gave identical
            // results and cost 14 %, profiles/round1_c/tf32x3_probe.txt).
            // Same byte offset, same swizzled position, so one descriptor
            // offset addresses either.
            for (int kb = 0; kb < t.num_kb; ++kb) {
                mbar_wait(smem_u32(full_bar + xs), xph);
                const u32 base = smem_u32(smem + xs * STAGE_BYTES);
                if (X3T) {
                    // A_lo -> TMEM: this thread's row (its TMEM lane), one
                    // 128-byte swizzle atom (32 fp32) at a time
                    const int row = quarter * 32 + lane;
#pragma unroll 1
                    for (int ka = 0; ka < KATOMS; ++ka) {
                        const u32 rbase = base + (u32)(ka * (BM_CTA * SWZ) + row * 128);
                        u32 l[32];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const u32 at = rbase + (u32)(((j ^ (row & 7)) & 7) * 16);
                            u32 x[4];
                            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "r"(at) : "memory");
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                l[4 * j + q] = __float_as_uint(__uint_as_float(x[q]) -
                                                               __uint_as_float(x[q] & 0xffffe000u));
                        }
                        const u32 taddr = tmem_base + ((u32)(quarter * 32) << 16) +
                                          (u32)(ALO_BASE + xs * ALO_COLS + ka * 32);
                        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
                                     "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                                     :: "r"(taddr), "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]),
                                        "r"(l[5]), "r"(l[6]), "r"(l[7]), "r"(l[8]), "r"(l[9]), "r"(l[10]),
                                        "r"(l[11]), "r"(l[12]), "r"(l[13]), "r"(l[14]), "r"(l[15]),
                                        "r"(l[16]), "r"(l[17]), "r"(l[18]), "r"(l[19]), "r"(l[20]),
                                        "r"(l[21]), "r"(l[22]), "r"(l[23]), "r"(l[24]), "r"(l[25]),
                                        "r"(l[26]), "r"(l[27]), "r"(l[28]), "r"(l[29]), "r"(l[30]), "r"(l[31])
                                     : "memory");
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    tc_fence_before();
                }
#pragma unroll 4
                for (int v = epi_tid + (X3T ? A_TILE / 16 : 0); v < LOAD_BYTES / 16; v += 128) {
                    const u32 at = base + (u32)v * 16u;
                    u32 x[4], h[4], l[4];
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "r"(at) : "memory");
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        h[q] = x[q] & 0xffffe000u;
                        l[q] = __float_as_uint(__uint_as_float(x[q]) - __uint_as_float(h[q]));
                    }
#ifdef OPEVO_X3_HI_INPLACE    // debug: write hi explicitly (the tensor core's own truncation
                    st_shared_v4(at, h[0], h[1], h[2], h[3]);   // gives the same results)
#endif
                    st_shared_v4(at + (u32)LO_OFF, l[0], l[1], l[2], l[3]);
                }
                fence_async_smem();                // generic smem writes -> the MMA (async proxy)
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(lo_bar + xs));
                if (++xs == STAGES) { xs = 0; xph ^= 1; }
            }
#endif
#if OPEVO_CONV
            const int w_tiles = geom.wo / TILE_W, h_tiles = geom.ho / TILE_H;
            const int w0 = (t.row_tile % w_tiles) * TILE_W;
            const int h0 = ((t.row_tile / w_tiles) % h_tiles) * TILE_H;
            const int n0 = (t.row_tile / (w_tiles * h_tiles)) * PAIR_TN + (int)prank * TILE_N;
            // tile row -> NHWC output pixel row (split-K paths); -1 for the
            // junk rows of padded lines
            auto out_row = [&](int lr) -> int {
                if (LINES) {
                    const int line = lr / LINE_ROWS, p = lr % LINE_ROWS;
                    if (p >= TILE_W || line >= TILE_N * TILE_H) return -1;
                    return ((n0 + line / TILE_H) * geom.ho + h0 + line % TILE_H) * geom.wo + w0 + p;
                }
                const int n = n0 + lr / (TILE_H * TILE_W);
                const int h = h0 + (lr / TILE_W) % TILE_H;
                const int w = w0 + lr % TILE_W;
                return (n * geom.ho + h) * geom.wo + w;
            };
#else
            const int row0 = t.row_tile * BM + (int)prank * BM_CTA;
            auto out_row = [&](int lr) -> int { return row0 + lr; };
#endif
            const u64 c_batch = (u64)t.batch * plane;
            mbar_wait(smem_u32(tfull_bar + buf), bph);
            tc_fence_after();
            if (epi_tid == 0 && eu < 5) UTRACE(2 + 3 * eu);
            if (first) {
                pdl_wait();                 // C may still be written by the previous launch
                if (epi_tid == 0) TRACE(6);
            }
            const u32 lane_addr = tmem_base + (u32)(buf * TMEM_USED) + ((u32)(quarter * 32) << 16);
            // drain the accumulator into registers, chunk by chunk; the last
            // chunk's TMEM load releases the buffer before its global stores
            auto release = [&]() {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2) mbar_arrive_cluster(tempty_leader0 + 8u * (u32)buf);
                    else         mbar_arrive(smem_u32(tempty_bar + buf));
                }
            };
            const int split = t.split;
            if (split == 1) {
                // TMEM -> registers -> swizzled smem chunk -> TMA store (one
                // bulk store per 32 x EPI_COLS chunk; two buffers per warp)
#pragma unroll 1
                for (int jm = 0; jm < MATOMS * BPU; ++jm) {
                    // jm: M atom (MATOMS > 1) or batch of the unit (BPU > 1)
                    const int ma = MATOMS > 1 ? jm : 0;
                    const int jb = BPU > 1 ? jm : 0;
                    const int lr0 = ma * 128 + quarter * 32;           // first tile row of the chunk
#pragma unroll 1
                    for (int c = 0; c < BN; c += STORE_COLS) {
                        float acc[STORE_COLS];
                        gather_acc<STORE_COLS>(lane_addr + jm * BN + c, acc);
                        if (first && c == 0 && epi_tid == 0) TRACE(12);
                        if (jm == MATOMS * BPU - 1 && c + STORE_COLS >= BN) release();
                        const u32 buf = epi_stage + (u32)((nchunk & 1) * EPI_BUF);
                        if (nchunk >= 2) {             // this buffer's previous store has read it
                            if (lane == 0) bulk_wait_read<1>();
                            __syncwarp();
                        }
                        stage_row(buf, lane, acc);
                        fence_async_smem();
                        __syncwarp();
                        if (lane == 0 && OPEVO_ABLATE != 6 && OPEVO_ABLATE != 7) {
#if OPEVO_CONV
                            if (LINES) {
                                // the chunk's 32 rows are 32 / LINE_ROWS padded
                                // lines: store their TILE_W valid pixels, skip the
                                // junk rows (direct st.global per lane measured
                                // no faster)
#pragma unroll
                                for (int q = 0; q < 32 / LINE_ROWS; ++q) {
                                    const int line = lr0 / LINE_ROWS + q;
                                    if (line >= TILE_N * TILE_H) break;   // rows past the tile's lines
                                    tma_store_4d(&tma_c, buf + (u32)(q * LINE_ROWS * EPI_ROW_BYTES), col0 + c, w0,
                                                 h0 + line % TILE_H, n0 + line / TILE_H);
                                }
                            } else {
                                const int n_l = lr0 / (TILE_H * TILE_W);
                                const int h_l = (lr0 / TILE_W) % TILE_H;
                                const int w_l = lr0 % TILE_W;
                                tma_store_4d(&tma_c, buf, col0 + c, w0 + w_l, h0 + h_l, n0 + n_l);
                            }
#elif OPEVO_BATCHED
                            tma_store_3d(&tma_c, buf, col0 + c, out_row(lr0), t.batch * BPU + jb);
#else
                            tma_store_2d(&tma_c, buf, col0 + c, out_row(lr0));
#endif
                            bulk_commit();
                        }
                        ++nchunk;
                        if (first && c == 0 && epi_tid == 0) TRACE(13);
                    }
                }
                if (first && epi_tid == 0) TRACE(7);
                if (epi_tid == 0 && eu < 5) UTRACE(3 + 3 * eu);
#if OPEVO_SPLIT_TMA > 1 && !OPEVO_CONV
            } else if (SPLITT > 1) {
                // ---- TMA split-K in one wave (the host guarantees every slice
                // of every tile is resident, so slice 0 may wait for the rest):
                // slices 1..S-1 publish their fp32 partial with TMA stores and
                // count in; slice 0 waits for S-1 arrivals, TMA-loads the
                // partials into its idle pipeline smem and sums them in z order
                // onto its own accumulator, then stores bf16 C.
                const int band0 = row0 + quarter * 32;          // first row of this warp's band
                u32* cnt = counters + (t.row_tile * sched.col_groups + t.col_tile);
                constexpr int CH = BN / 32;                      // 32-column fp32 chunks
                if (t.kz != 0) {
                    const u32 wst = smem_u32(smem) + (u32)(quarter * CH * 4096);
#pragma unroll 1
                    for (int c = 0; c < CH; ++c) {
                        float acc[32];
                        gather_acc<32>(lane_addr + c * 32, acc);
                        stage_row_f32(wst + (u32)(c * 4096), lane, acc);
                    }
                    release();
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        for (int c = 0; c < CH; ++c) tma_store_3d(&tma_w, wst + (u32)(c * 4096), col0 + c * 32, band0, t.kz);
                        bulk_commit();
                        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // written, not just read
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    epi_bar();
                    if (epi_tid == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(cnt) : "memory");
                } else {
                    if (lane == 0) {
                        const u64 t0 = global_ns();
                        while (ld_acquire_gpu(cnt) < (u32)(SPLITT - 1)) {
                            __nanosleep(64);
                            if (global_ns() - t0 > 4000000000ull) asm volatile("trap;");
                        }
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        const u32 pb = smem_u32(smem) + (u32)(quarter * (SPLITT - 1) * CH * 4096);
                        // single lane: the plain arrive (mbar_expect_tx elects within a full warp)
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                                     :: "r"(smem_u32(part_bar + quarter)), "r"((u32)((SPLITT - 1) * CH * 4096))
                                     : "memory");
                        for (int z = 1; z < SPLITT; ++z)
                            for (int c = 0; c < CH; ++c)
                                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                                             "[%0], [%1, {%3, %4, %5}], [%2];"
                                             :: "r"(pb + (u32)(((z - 1) * CH + c) * 4096)), "l"(&tma_w),
                                                "r"(smem_u32(part_bar + quarter)), "r"(col0 + c * 32), "r"(band0), "r"(z)
                                             : "memory");
                    }
                    __syncwarp();
                    mbar_wait(smem_u32(part_bar + quarter), 0);
                    epi_bar();
                    if (epi_tid == 0) *cnt = 0u;                     // ready for the next launch
                    const u32 pb = smem_u32(smem) + (u32)(quarter * (SPLITT - 1) * CH * 4096);
#pragma unroll 1
                    for (int c = 0; c < BN; c += STORE_COLS) {
                        float acc[STORE_COLS];
                        gather_acc<STORE_COLS>(lane_addr + c, acc);
                        if (c + STORE_COLS >= BN) release();
#pragma unroll
                        for (int h = 0; h < STORE_COLS / 32; ++h)
                            for (int z = 1; z < SPLITT; ++z)
                                add_row_f32(pb + (u32)(((z - 1) * CH + c / 32 + h) * 4096), lane, acc + 32 * h);
                        const u32 buf = epi_stage + (u32)((nchunk & 1) * EPI_BUF);
                        if (nchunk >= 2) {
                            if (lane == 0) bulk_wait_read<1>();
                            __syncwarp();
                        }
                        stage_row(buf, lane, acc);
                        fence_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tma_c, buf, col0 + c, band0);
                            bulk_commit();
                        }
                        ++nchunk;
                    }
                }
#endif
            } else if (SPLITCL > 1) {
                // ---- DSMEM split-K: this CTA is slice kz == cluster rank
                float* own = reinterpret_cast<float*>(smem);
                // 1. TMEM -> own partial in shared memory (row-major [BM][BN])
#pragma unroll 1
                for (int c = 0; c < BN; c += EPI_COLS) {
                    float acc[EPI_COLS];
                    const int lr = quarter * 32 + lane;
                    gather_acc(lane_addr + c, acc);
                    float* dst = own + lr * RED_LD + c;
#pragma unroll
                    for (int j = 0; j < EPI_COLS; j += 4)
                        *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
                }
                release();
                if (epi_tid == 0) TRACE(12);
                // generic-proxy smem writes -> visible to the bulk-copy (async) proxy
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                epi_bar();
            }
            if (SPLITCL > 1 || SPLITT > 1) {
                // DSMEM: steps 2-4 (exchange + reduction) run after the role
                // loops with every thread of the CTA, see below; TMA: done above
            } else if (split > 1) {
                // split-K: publish this slice's fp32 partial, count arrivals; the
                // last CTA of the tile sums all slices in z order (its own from
                // TMEM, the rest from L2) and writes the output
#pragma unroll 1
                for (int ma = 0; ma < MATOMS; ++ma) {
                    const int r = out_row(ma * 128 + quarter * 32 + lane);
#pragma unroll 1
                    for (int c = 0; c < BN; c += EPI_COLS) {
                        float acc[EPI_COLS];
                        gather_acc(lane_addr + ma * BN + c, acc);      // warp-collective
                        if (r < 0) continue;                           // junk row of a padded line
                        float* dst = ws + (u64)t.kz * slice + c_batch + (u64)r * cols + col0 + c;
#pragma unroll
                        for (int j = 0; j < EPI_COLS; j += 4)
                            st_v4(dst + j, __float_as_uint(acc[j]), __float_as_uint(acc[j + 1]),
                                  __float_as_uint(acc[j + 2]), __float_as_uint(acc[j + 3]));
                    }
                }
                epi_bar();                  // all partial stores issued (CTA scope)
                if (epi_tid == 0) {
                    const u32 tile = (u32)((((t.batch * sched.row_tiles + t.row_tile) * sched.col_groups
                                            + t.col_tile / CLUSTER) * CLSZ) + crank);
                    // release: cumulative over the CTA's partial stores ordered by the barrier
                    const u32 prev = atom_add_release_gpu(counters + tile, 1u);
                    const u32 last = (prev == (u32)(split - 1)) ? 1u : 0u;
                    if (last) {
                        fence_acq_rel_gpu();            // acquire the other slices' partials
                        counters[tile] = 0u;            // ready for the next launch
                    }
                    *last_flag = last;
                }
                epi_bar();
                if (*last_flag) {
#pragma unroll 1
                    for (int ma = 0; ma < MATOMS; ++ma) {
                        const int r = out_row(ma * 128 + quarter * 32 + lane);
#pragma unroll 1
                        for (int c = 0; c < BN; c += EPI_COLS) {
                            float own[EPI_COLS], acc[EPI_COLS];
                            gather_acc(lane_addr + ma * BN + c, own);  // warp-collective
                            if (r < 0) continue;                       // junk row of a padded line
#pragma unroll
                            for (int j = 0; j < EPI_COLS; ++j) acc[j] = 0.0f;
                            const u64 base = c_batch + (u64)r * cols + col0 + c;
                            // two slices in flight per step; summation order is z = 0..split-1
                            for (int z = 0; z < split; z += 2) {
                                float4 p0[EPI_COLS / 4], p1[EPI_COLS / 4];
                                const bool use1 = z + 1 < split;
                                if (z != t.kz) {
                                    const float* src = ws + (u64)z * slice + base;
#pragma unroll
                                    for (int j = 0; j < EPI_COLS / 4; ++j) p0[j] = ld_cg_f4(src + 4 * j);
                                }
                                if (use1 && z + 1 != t.kz) {
                                    const float* src = ws + (u64)(z + 1) * slice + base;
#pragma unroll
                                    for (int j = 0; j < EPI_COLS / 4; ++j) p1[j] = ld_cg_f4(src + 4 * j);
                                }
#pragma unroll
                                for (int j = 0; j < EPI_COLS / 4; ++j) {
                                    if (z == t.kz) {
                                        acc[4 * j] += own[4 * j]; acc[4 * j + 1] += own[4 * j + 1];
                                        acc[4 * j + 2] += own[4 * j + 2]; acc[4 * j + 3] += own[4 * j + 3];
                                    } else {
                                        acc[4 * j] += p0[j].x; acc[4 * j + 1] += p0[j].y;
                                        acc[4 * j + 2] += p0[j].z; acc[4 * j + 3] += p0[j].w;
                                    }
                                }
                                if (use1) {
#pragma unroll
                                    for (int j = 0; j < EPI_COLS / 4; ++j) {
                                        if (z + 1 == t.kz) {
                                            acc[4 * j] += own[4 * j]; acc[4 * j + 1] += own[4 * j + 1];
                                            acc[4 * j + 2] += own[4 * j + 2]; acc[4 * j + 3] += own[4 * j + 3];
                                        } else {
                                            acc[4 * j] += p1[j].x; acc[4 * j + 1] += p1[j].y;
                                            acc[4 * j + 2] += p1[j].z; acc[4 * j + 3] += p1[j].w;
                                        }
                                    }
                                }
                            }
                            store_row(c_out, base, acc);
                        }
                    }
                }
                release();                  // TMEM buffer (kept for the own-slice read)
                epi_bar();                  // last_flag is reused by the next unit
            }
            first = false;
            ++eu;
            if (++buf == NBUF) { buf = 0; bph ^= 1; }
        }
        // staged chunks must be read out before the CTA's smem goes away
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
    }

    tc_fence_before();
    __syncthreads();
#if OPEVO_SPLIT_CLUSTER > 1
    {
        // ---- DSMEM split-K reduction (one unit per cluster; slice kz == rank)
        // 2. every slice has staged its partial and finished its mainloop
        cluster_sync();
        if (threadIdx.x == 0) TRACE(13);
        const float* own = reinterpret_cast<const float*>(smem);
        if (threadIdx.x == 0) {
            // push the row block each peer owns into that peer's RECV slot
            for (int z = 0; z < SPLITCL; ++z) {
                if (z == (int)crank) continue;
                const int slot = (int)crank < z ? (int)crank : (int)crank - 1;
                const u32 dst = mapa_cta(smem_u32(smem + RED_OWN_BYTES + slot * RED_BLOCK_BYTES), (u32)z);
                const u32 bar = mapa_cta(smem_u32(red_bar), (u32)z);
                asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes "
                             "[%0], [%1], %2, [%3];"
                             :: "r"(dst), "r"(smem_u32(own + z * RED_ROWS * RED_LD)),
                                "r"((u32)RED_BLOCK_BYTES), "r"(bar) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        // 3. the peers' blocks of my rows have landed: sum in z order, write
        mbar_wait(smem_u32(red_bar), 0);
        if (threadIdx.x == 0) TRACE(14);
        const Unit t = decode(u_first);
        const int col0 = t.col_tile * BN;
        const u64 c_batch = (u64)t.batch * (u64)rows * (u64)cols;
#if OPEVO_CONV
        const int w_tiles = geom.wo / TILE_W, h_tiles = geom.ho / TILE_H;
        const int w0 = (t.row_tile % w_tiles) * TILE_W;
        const int h0 = ((t.row_tile / w_tiles) % h_tiles) * TILE_H;
        const int n0 = (t.row_tile / (w_tiles * h_tiles)) * PAIR_TN;
#endif
        const float* recv = reinterpret_cast<const float*>(smem + RED_OWN_BYTES);
        const int my_row0 = (int)crank * RED_ROWS;
        constexpr int SEGS = BN / 8;                     // 8 outputs per thread-step
#pragma unroll 1
        for (int e = threadIdx.x; e < RED_ROWS * SEGS; e += NUM_THREADS) {
            const int rr = e / SEGS, c8 = (e - rr * SEGS) * 8;
            float acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
            for (int z = 0; z < SPLITCL; ++z) {
                const float* src = (z == (int)crank)
                    ? own + (my_row0 + rr) * RED_LD + c8
                    : recv + ((z < (int)crank ? z : z - 1) * RED_ROWS + rr) * RED_LD + c8;
                const float4 x = *reinterpret_cast<const float4*>(src);
                const float4 y = *reinterpret_cast<const float4*>(src + 4);
                acc[0] += x.x; acc[1] += x.y; acc[2] += x.z; acc[3] += x.w;
                acc[4] += y.x; acc[5] += y.y; acc[6] += y.z; acc[7] += y.w;
            }
            const int lr = my_row0 + rr;
#if OPEVO_CONV
            const int r = (n0 + lr / (TILE_H * TILE_W)) * geom.ho * geom.wo +
                          (h0 + (lr / TILE_W) % TILE_H) * geom.wo + (w0 + lr % TILE_W);
#else
            const int r = t.row_tile * BM + lr;
#endif
#if OPEVO_OUT_F32
            float* dst = reinterpret_cast<float*>(c_out) + c_batch + (u64)r * cols + col0 + c8;
            st_v4(dst, __float_as_uint(acc[0]), __float_as_uint(acc[1]),
                  __float_as_uint(acc[2]), __float_as_uint(acc[3]));
            st_v4(dst + 4, __float_as_uint(acc[4]), __float_as_uint(acc[5]),
                  __float_as_uint(acc[6]), __float_as_uint(acc[7]));
#else
            u16* dst = reinterpret_cast<u16*>(c_out) + c_batch + (u64)r * cols + col0 + c8;
            st_v4(dst, pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]),
                  pack_bf16(acc[4], acc[5]), pack_bf16(acc[6], acc[7]));
#endif
        }
        if (threadIdx.x == 0) TRACE(7);
        // 4. my outgoing copies have finished reading `own`
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
    }
#endif
    if (threadIdx.x == 0) TRACE(8);
    if (CLSZ > 1) cluster_sync();
    if (threadIdx.x == 0) TRACE(15);
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;"
                         :: "r"(tmem_base), "r"(TMEM_ALLOC) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                         :: "r"(tmem_base), "r"(TMEM_ALLOC) : "memory");
    }
}
