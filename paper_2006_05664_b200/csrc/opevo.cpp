// libopevo: the C-ABI trial evaluator (see include/opevo.h).
//
// Replaces the reference's evaluation seam (pkg/src/topotune/engine.py:264-290,
// benchmarks.py:278-302): one call per configuration compiles (NVRTC, cached),
// verifies and CUDA-event-times a hand-written sm_100a kernel.
//
// libcuda and libnvrtc are dlopen'ed on first use, so the library loads (and
// its compile-only entry point works) on a machine without a GPU.

#include "opevo.h"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <thread>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <unistd.h>
#include <unordered_map>
#include <vector>

extern "C" const unsigned char opevo_util_cubin[];
extern "C" const size_t opevo_util_cubin_len;
extern "C" const char opevo_gemm_source[];
extern "C" const char opevo_sgemm_source[];

namespace {

// ------------------------------------------------------------------ errors
void put_err(char* err, size_t len, const char* fmt, ...) {
    if (!err || len == 0) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, len, fmt, ap);
    va_end(ap);
}

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------- libcuda
struct Driver {
#define OPEVO_CU_FN(name, sym) decltype(&::sym) name = nullptr;
#define OPEVO_CU_LIST(X)                                          \
    X(Init, cuInit)                                               \
    X(DeviceGet, cuDeviceGet)                                     \
    X(DeviceGetAttribute, cuDeviceGetAttribute)                   \
    X(PrimaryCtxRetain, cuDevicePrimaryCtxRetain)                 \
    X(PrimaryCtxRelease, cuDevicePrimaryCtxRelease_v2)            \
    X(CtxSetCurrent, cuCtxSetCurrent)                             \
    X(CtxSynchronize, cuCtxSynchronize)                           \
    X(ModuleLoadData, cuModuleLoadData)                           \
    X(ModuleUnload, cuModuleUnload)                               \
    X(ModuleGetFunction, cuModuleGetFunction)                     \
    X(FuncLoad, cuFuncLoad)                                       \
    X(FuncSetAttribute, cuFuncSetAttribute)                       \
    X(FuncGetAttribute, cuFuncGetAttribute)                       \
    X(LaunchKernel, cuLaunchKernel)                               \
    X(LaunchKernelEx, cuLaunchKernelEx)                           \
    X(MemAlloc, cuMemAlloc_v2)                                    \
    X(MemFree, cuMemFree_v2)                                      \
    X(MemAllocHost, cuMemAllocHost_v2)                            \
    X(MemFreeHost, cuMemFreeHost)                                 \
    X(MemHostAlloc, cuMemHostAlloc)                               \
    X(MemHostGetDevicePointer, cuMemHostGetDevicePointer_v2)      \
    X(MemcpyHtoD, cuMemcpyHtoD_v2)                                \
    X(MemcpyDtoH, cuMemcpyDtoH_v2)                                \
    X(MemcpyHtoDAsync, cuMemcpyHtoDAsync_v2)                      \
    X(MemcpyDtoHAsync, cuMemcpyDtoHAsync_v2)                      \
    X(MemsetD8, cuMemsetD8_v2)                                    \
    X(MemsetD8Async, cuMemsetD8Async)                             \
    X(StreamCreate, cuStreamCreate)                               \
    X(StreamDestroy, cuStreamDestroy_v2)                          \
    X(StreamSynchronize, cuStreamSynchronize)                     \
    X(StreamBeginCapture, cuStreamBeginCapture_v2)                \
    X(StreamEndCapture, cuStreamEndCapture)                       \
    X(GraphInstantiate, cuGraphInstantiateWithFlags)              \
    X(GraphLaunch, cuGraphLaunch)                                 \
    X(GraphUpload, cuGraphUpload)                                 \
    X(GraphExecDestroy, cuGraphExecDestroy)                       \
    X(GraphDestroy, cuGraphDestroy)                               \
    X(EventCreate, cuEventCreate)                                 \
    X(EventDestroy, cuEventDestroy_v2)                            \
    X(EventRecord, cuEventRecord)                                 \
    X(EventSynchronize, cuEventSynchronize)                       \
    X(EventElapsedTime, cuEventElapsedTime)                       \
    X(TensorMapEncodeTiled, cuTensorMapEncodeTiled)               \
    X(OccupancyMaxBlocks, cuOccupancyMaxActiveBlocksPerMultiprocessor) \
    X(GetErrorString, cuGetErrorString)                           \
    X(GetErrorName, cuGetErrorName)
    OPEVO_CU_LIST(OPEVO_CU_FN)
    void* handle = nullptr;
    bool ok = false;
    std::string why;
};

Driver g_cu;
std::once_flag g_cu_once;

void load_driver() {
    std::call_once(g_cu_once, [] {
        g_cu.handle = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        if (!g_cu.handle) g_cu.handle = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
        if (!g_cu.handle) {
            g_cu.why = std::string("cannot dlopen libcuda.so.1: ") + dlerror();
            return;
        }
#define OPEVO_CU_LOAD(name, sym)                                                     \
    g_cu.name = reinterpret_cast<decltype(g_cu.name)>(dlsym(g_cu.handle, #sym));    \
    if (!g_cu.name) { g_cu.why = "libcuda lacks " #sym; return; }
        OPEVO_CU_LIST(OPEVO_CU_LOAD)
        CUresult r = g_cu.Init(0);
        if (r != CUDA_SUCCESS) {
            g_cu.why = "cuInit failed (" + std::to_string((int)r) + ")";
            return;
        }
        g_cu.ok = true;
    });
}

const char* cu_str(CUresult r) {
    const char* s = nullptr;
    if (g_cu.GetErrorString) g_cu.GetErrorString(r, &s);
    return s ? s : "unknown CUDA error";
}

// Errors after which the context is unusable (the worker must restart).
bool is_sticky(CUresult r) {
    return (r >= 700 && r <= 720) || r == CUDA_ERROR_UNKNOWN || r == CUDA_ERROR_CONTEXT_IS_DESTROYED;
}

// ------------------------------------------------------------- libnvrtc
struct Nvrtc {
#define OPEVO_RTC_LIST(X)                              \
    X(Create, nvrtcCreateProgram)                      \
    X(Compile, nvrtcCompileProgram)                    \
    X(Destroy, nvrtcDestroyProgram)                    \
    X(GetCUBINSize, nvrtcGetCUBINSize)                 \
    X(GetCUBIN, nvrtcGetCUBIN)                         \
    X(GetLogSize, nvrtcGetProgramLogSize)              \
    X(GetLog, nvrtcGetProgramLog)                      \
    X(ErrorString, nvrtcGetErrorString)                \
    X(Version, nvrtcVersion)
    OPEVO_RTC_LIST(OPEVO_CU_FN)
    void* handle = nullptr;
    bool ok = false;
    std::string why;
    int major = 0, minor = 0;
};

Nvrtc g_rtc;
std::once_flag g_rtc_once;

void load_nvrtc() {
    std::call_once(g_rtc_once, [] {
        const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
        for (const char* n : names) {
            g_rtc.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (g_rtc.handle) break;
        }
        if (!g_rtc.handle) {
            g_rtc.why = "cannot dlopen libnvrtc.so.12";
            return;
        }
#define OPEVO_RTC_LOAD(name, sym)                                                     \
    g_rtc.name = reinterpret_cast<decltype(g_rtc.name)>(dlsym(g_rtc.handle, #sym));  \
    if (!g_rtc.name) { g_rtc.why = "libnvrtc lacks " #sym; return; }
        OPEVO_RTC_LIST(OPEVO_RTC_LOAD)
        g_rtc.Version(&g_rtc.major, &g_rtc.minor);
        g_rtc.ok = true;
    });
}

// ------------------------------------------------------------- knobs
struct Knobs {
    int bm, bn, bk, stages, split, cluster, tile_h, tile_w, acc, cg, grid_mode, b_res, bpu, line;
};

Knobs read_knobs(const int32_t* k, int n) {
    int32_t v[OPEVO_NUM_KNOBS] = {128, 128, 64, 4, 1, 1, 1, 1, 1, 1, 0, 0, 1, 0};
    for (int i = 0; i < n && i < OPEVO_NUM_KNOBS; ++i) v[i] = k[i];
    return Knobs{v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9], v[10], v[11], v[12], v[13]};
}

// Family 3 (fp32 GEMM as 3xTF32 on tcgen05) takes BK in fp32 elements at the
// ABI; inside the library -- cache key, NVRTC macros, shared-memory sizing,
// tensor maps -- each fp32 operand is viewed as bf16 pairs, so BK and K are
// counted in bf16 units (twice the fp32 count).
constexpr int FAMILY_X3 = 3;
Knobs lib_knobs(int family, const int32_t* k, int n) {
    Knobs kn = read_knobs(k, n);
    if (family == FAMILY_X3) kn.bk *= 2;
    return kn;
}

// Kernel family of an operator: 0 bf16 GEMM, 1 conv, 2 fp32 SIMT, 3 fp32 3xTF32.
int family_of(const opevo_op_desc& d) {
    if (d.kind == OPEVO_CONV2D) return 1;
    return d.dtype == OPEVO_F32 ? 2 : d.dtype == OPEVO_F32_TF32X3 ? FAMILY_X3 : 0;
}

// Tile rows one CTA holds (a CTA pair splits BM in two) and the MMA atoms
// per K step (mirror BM_CTA / MATOMS in gemm_sm100.cuh).
int bm_cta_of(const Knobs& k) { return k.cg == 2 ? k.bm / 2 : k.bm; }
int matoms_of(const Knobs& k) { return bm_cta_of(k) == 256 ? 2 : 1; }

// TMEM columns the kernel allocates (two accumulator buffers when they fit;
// 3xTF32 single-CTA 128-row tiles with 128-byte swizzle add the A_lo ring,
// mirrors X3T / TMEM_NEED).
int tmem_alloc_cols(const Knobs& k, int family = 0) {
    const int used = matoms_of(k) * k.bn * k.acc * std::max(1, k.bpu);
    const int nbuf = 4 * used <= 256 ? 4 : 2 * used <= 512 ? 2 : 1;   // mirrors NBUF
    int want = nbuf * used;
    const int alo = k.bk / 2 * k.stages;                                 // k.bk in bf16 units here
    if (family == FAMILY_X3 && k.cg == 1 && k.bm == 128 && k.bk >= 64 && want + alo <= 512 &&
        !(getenv("OPEVO_EXTRA_FLAGS") && strstr(getenv("OPEVO_EXTRA_FLAGS"), "OPEVO_X3_SMEM_ALO=1")))
        want += alo;
    int cols = 32;
    while (cols < want) cols *= 2;
    return cols;
}

int swizzle_bytes(int bk) { return bk * 2 >= 128 ? 128 : bk * 2; }

// Weight-resident conv (knob b_res): the whole BN x K weight panel is loaded
// once per CTA into shared memory (one TMA box of the atom view), so the
// pipeline stages carry only the activation tile.  128-byte swizzle (BK a
// multiple of 64) and no split over taps.
bool b_resident(const Knobs& k, int family) {
    return family == 1 && k.b_res && k.bk % 64 == 0 && k.split == 1;
}

// Conv "halo lines" (OPEVO_HALO in gemm_sm100.cuh): a conv tile whose width
// does not divide BM is read as lines of TILE_W = 17 - KW output pixels padded
// to 16 tile rows; one TMA box per filter row serves its KW taps.  Returns KW,
// or 0 for the one-box-per-tap layout.
int halo_kw(const Knobs& k, int family) {
    const int bm_cta = bm_cta_of(k);
    return (family == 1 && k.line == 0 && k.tile_w >= 1 && k.tile_w < 16 && k.tile_h >= 1 &&
            bm_cta % (k.tile_h * k.tile_w) != 0)
               ? 17 - k.tile_w : 0;
}

// K-fused operand loads (GEMM family, 128-byte swizzle, no multicast slices):
// mirrors FUSED_K in gemm_sm100.cuh.
bool fused_k(const Knobs& k) { return swizzle_bytes(k.bk) == 128 && k.cluster == 1; }

// DSMEM split-K (the split slices of a tile form a cluster and reduce in
// shared memory) when the shape allows it; split is then compiled in.
size_t dsmem_red_bytes(const Knobs& k) {
    const int s = k.split, ld = k.bn + 4;   // rows padded by 16 B (bank conflicts)
    return (size_t)k.bm * ld * 4 + (size_t)(s - 1) * (k.bm / s) * ld * 4;
}

size_t wide_epi_stage_bytes(const Knobs& k, int out_f32);

// TMA split-K (split 2 or 4 on single-CTA 128-row bf16 GEMM tiles): the
// slices of a tile reduce through fp32 partials in global memory written
// and read by TMA, slice 0 waiting for the others -- one wave only (checked
// at bind time).  Mirrors SPLITT in gemm_sm100.cuh and tma_split in mapping.py.
int tma_split(const Knobs& k, int family, int batched) {
    return (family == 0 && !batched && (k.split == 2 || k.split == 4) && k.cg == 1 && k.cluster == 1 &&
            k.bm == 128 && k.acc == 1 && k.bpu <= 1 && k.bn % 32 == 0 &&
            (size_t)(k.split - 1) * 128 * k.bn * 4 <= 196608)
               ? k.split : 0;
}

bool dsmem_split(const Knobs& k, int family, int batched = 0) {
    return family != 2 && (k.split == 2 || k.split == 4 || k.split == 8) && k.cg == 1 &&
           !(family == 1 && k.line) &&   // padded lines reduce through the global path
           k.cluster == 1 && k.bm == 128 && !tma_split(k, family, batched) &&
           (dsmem_red_bytes(k) + 1023) / 1024 * 1024 + wide_epi_stage_bytes(k, family == FAMILY_X3) + 1024 + 256 <=
               232448;
}

// TMA-store epilogue chunk width before the two-CTAs-per-SM rule below.
int wide_epi_cols(const Knobs& k, int out_f32) {
    return (!out_f32 && k.bn % 64 == 0 && k.acc == 1) ? 64 : k.bn % 32 == 0 ? 32 : 16;
}

// TMA-store staging: 4 epilogue warps x 2 buffers x 32 rows x STORE_COLS outputs.
size_t epi_stage_bytes_cols(int cols, int out_f32) { return (size_t)4 * 2 * 32 * cols * (out_f32 ? 4 : 2); }
size_t wide_epi_stage_bytes(const Knobs& k, int out_f32) {
    return epi_stage_bytes_cols(wide_epi_cols(k, out_f32), out_f32);
}

// Pipeline (operand stages or split-K reduction buffer) of one CTA, 1 KB aligned:
// a CTA pair stages BM/2 rows of A and BN/2 rows of B each (mirrors PIPE_BYTES).
size_t pipe_bytes(const Knobs& k, int family, int batched) {
    const int a_rows = bm_cta_of(k);
    const int b_rows = b_resident(k, family) ? 0 : k.bn / (k.cg == 2 ? 2 : 1) * std::max(1, halo_kw(k, family));
    size_t pipe = (size_t)k.stages * (size_t)(a_rows + b_rows) * (size_t)k.bk * 2 * (size_t)std::max(1, k.bpu);
    if (family == FAMILY_X3) pipe *= 2;       // hi (as landed) + lo parts per stage
    if (dsmem_split(k, family, batched)) pipe = std::max(pipe, dsmem_red_bytes(k));
    if (const int ts = tma_split(k, family, batched))
        pipe = std::max(pipe, (size_t)std::max(ts - 1, 1) * 128 * k.bn * 4);   // SPLITT_BYTES
    return (pipe + 1023) / 1024 * 1024;
}

// Two CTAs per SM need 2 x (dynamic smem + the 1 KB per-CTA reservation) within
// the SM's 228 KB.  A single-CTA or CTA-pair bf16 instance that misses this only by its
// 64-column epilogue staging (32 KB) stages 32 columns instead (16 KB): one
// more TMEM load / fence / store per 64 columns, in exchange for a second CTA
// -- i.e. a second MMA-issuing warp -- on every SM (conv halo tiles with 2
// stages; profiles/round2/two_ctas_per_sm.txt).  Not for resident weight
// panels (the panel alone keeps them at one CTA) nor for accumulators that
// take more than half of TMEM.  OPEVO_NARROW_EPI=0 disables
// the rule (A/B experiments).  Mirrors Knobs.narrow_epi in mapping.py.
constexpr size_t SM_SMEM_BYTES = 233472, CTA_RESERVED_SMEM = 1024;
bool narrow_epi(const Knobs& k, int family, int out_f32, int batched) {
    static const bool enabled = !(getenv("OPEVO_NARROW_EPI") && getenv("OPEVO_NARROW_EPI")[0] == '0');
    if (!enabled || (family != 0 && family != 1) || out_f32 || wide_epi_cols(k, out_f32) != 64 ||
        k.cluster != 1 || dsmem_split(k, family, batched) || b_resident(k, family) || tmem_alloc_cols(k) > 256)
        return false;
    const size_t base = pipe_bytes(k, family, batched) + 1024 + 256 + CTA_RESERVED_SMEM;
    return 2 * (base + epi_stage_bytes_cols(64, 0)) > SM_SMEM_BYTES &&
           2 * (base + epi_stage_bytes_cols(32, 0)) <= SM_SMEM_BYTES;
}

// TMA-store epilogue chunk width (mirrors STORE_COLS in gemm_sm100.cuh).
int epi_cols(const Knobs& k, int family, int out_f32, int batched) {
    return narrow_epi(k, family, out_f32, batched) ? 32 : wide_epi_cols(k, out_f32);
}

// per-CTA: the pipeline, then the epilogue staging (1024-aligned) and the
// barriers (mirrors EPI_OFF/BAR_OFF)
size_t smem_bytes(const Knobs& k, int family = 0, int out_f32 = 0, int batched = 0) {
    if (family == 2) return 0;
    return pipe_bytes(k, family, batched) + epi_stage_bytes_cols(epi_cols(k, family, out_f32, batched), out_f32) +
           1024 + 256;
}

uint64_t fnv1a(const char* s, size_t n, uint64_t h = 1469598103934665603ull) {
    for (size_t i = 0; i < n; ++i) { h ^= (unsigned char)s[i]; h *= 1099511628211ull; }
    return h;
}

// Everything that changes the generated code is in the key; split-K is a
// launch parameter and is not.
// -lineinfo (for ncu source views) triples the cubin size; opt in with
// OPEVO_LINEINFO=1.  It is part of the cache key.
bool want_lineinfo() {
    const char* v = getenv("OPEVO_LINEINFO");
    return v && v[0] == '1';
}

// Extra -D flags for debug instances (e.g. "-DOPEVO_TRACE=1"); part of the key.
std::string extra_flags() {
    const char* v = getenv("OPEVO_EXTRA_FLAGS");
    return v ? v : "";
}

// Fault injection for the robustness tests (OPEVO_FAULT_KNOBS="bm,bn,bk,..."):
// an instance whose knob vector starts with these values is compiled with
// OPEVO_ABLATE=5, a `trap` at kernel entry -- the sticky fault that poisons
// a CUDA context, as a broken candidate would.  Part of the cache key.
std::string instance_flags(int family, const Knobs& k) {
    std::string f = extra_flags();
    const char* v = getenv("OPEVO_FAULT_KNOBS");
    if (!v || !*v || family == 2) return f;
    const int kv[OPEVO_NUM_KNOBS] = {k.bm, k.bn, k.bk, k.stages, k.split, k.cluster, k.tile_h, k.tile_w,
                                     k.acc, k.cg, k.grid_mode, k.b_res, k.bpu, k.line};
    std::istringstream in(v);
    std::string tok;
    int i = 0;
    while (std::getline(in, tok, ',')) {
        if (i >= OPEVO_NUM_KNOBS || atoi(tok.c_str()) != kv[i]) return f;
        ++i;
    }
    return i ? f + " -DOPEVO_ABLATE=5" : f;
}

bool want_pdl() {
    const char* v = getenv("OPEVO_NO_PDL");
    return !(v && v[0] == '1');
}

std::string make_key(int family, const Knobs& k, int batched, int out_f32) {
    static const uint64_t src_hash = fnv1a(opevo_gemm_source, strlen(opevo_gemm_source));
    static const uint64_t simt_hash = fnv1a(opevo_sgemm_source, strlen(opevo_sgemm_source));
    const std::string extra = instance_flags(family, k);
    const uint64_t h = fnv1a(extra.data(), extra.size(), family == 2 ? simt_hash : src_hash);
    char buf[256];
    if (family == 2) {
        // fp32 SIMT family: slots 0..7 hold (n2, n3, n4, m2, m3, m4, k2, k3)
        snprintf(buf, sizeof buf, "f2_n%d.%d.%d_m%d.%d.%d_k%d.%d_b%d_%s%012llx", k.bm, k.bn, k.bk,
                 k.stages, k.split, k.cluster, k.tile_h, k.tile_w, batched,
                 want_lineinfo() ? "L" : "", (unsigned long long)(h & 0xffffffffffffull));
        return buf;
    }
    char line[16] = "";
    if (family == 1 && k.line) snprintf(line, sizeof line, "_l%d", k.line);
    snprintf(buf, sizeof buf, "f%d_m%d_n%d_k%d_s%d_b%d_o%d_c%d_h%d_w%d_a%d_g%d%s%s%s_%s%012llx", family,
             k.bm, k.bn, k.bk, k.stages, batched, out_f32, k.cluster, family == 1 ? k.tile_h : 1,
             family == 1 ? k.tile_w : 1, k.acc,
             k.cg * 100 + (dsmem_split(k, family, batched) ? k.split : 0) + 10 * tma_split(k, family, batched),
             b_resident(k, family) ? "_r" : k.bpu > 1 ? (k.bpu == 2 ? "_u2" : "_u4") : "", line,
             narrow_epi(k, family, out_f32, batched) ? "_e32" : "",
             want_lineinfo() ? "L" : "",
             (unsigned long long)(h & 0xffffffffffffull));
    return buf;
}

// fp32 SIMT family geometry from the knob slots (n2,n3,n4,m2,m3,m4,k2,k3).
struct Simt {
    int n2, n3, n4, m2, m3, m4, k2, k3;
    int threads() const { return n3 * m3; }
    int bm() const { return n2 * n3 * n4; }
    int bn() const { return m2 * m3 * m4; }
    int ks() const { return k2 * k3; }
    size_t smem() const { return (size_t)ks() * (size_t)(bm() + bn() + 2) * 4; }
};

Simt simt_of(const Knobs& k) {
    return Simt{k.bm, k.bn, k.bk, k.stages, k.split, k.cluster, k.tile_h, k.tile_w};
}

// Structural checks shared by compile and bind (operator-independent).
bool knobs_compilable(int family, const Knobs& k, char* err, size_t len) {
    if (family == 2) {
        const Simt g = simt_of(k);
        const int f[8] = {g.n2, g.n3, g.n4, g.m2, g.m3, g.m4, g.k2, g.k3};
        for (int v : f)
            if (v < 1) {
                put_err(err, len, "SIMT factors must be >= 1");
                return false;
            }
        if (g.threads() > 1024) {
            put_err(err, len, "n3*m3 = %d threads per block exceeds 1024", g.threads());
            return false;
        }
        if (g.n2 * g.n4 * g.m2 * g.m4 > 256) {
            put_err(err, len, "per-thread tile %dx%d exceeds the register file",
                    g.n2 * g.n4, g.m2 * g.m4);
            return false;
        }
        if (g.k3 > 64 || g.smem() > 232448) {
            put_err(err, len, "shared tile %zu B (k3=%d) too large", g.smem(), g.k3);
            return false;
        }
        return true;
    }
    if (!(k.bm == 128 || k.bm == 256 || (k.bm == 512 && k.cg == 2 && halo_kw(k, family)))) {
        put_err(err, len, "BM=%d unsupported (128 or 256; 512 for a halo-line conv CTA pair)", k.bm);
        return false;
    }
    if (k.bn < 16 || k.bn > 256 || k.bn % 16) {
        put_err(err, len, "BN=%d must be a multiple of 16 in [16,256]", k.bn);
        return false;
    }
    const bool bk_ok = k.bk == 16 || k.bk == 32 || (k.bk >= 64 && k.bk <= 256 && k.bk % 64 == 0);
    if (!bk_ok) {
        put_err(err, len, "BK=%d unsupported (16, 32 or a multiple of 64 up to 256)", k.bk);
        return false;
    }
    if (k.stages < 1 || k.stages > 16) {
        put_err(err, len, "stages=%d out of range", k.stages);
        return false;
    }
    // the split-K workspace is allocated for OPEVO_MAX_SPLIT slices when the
    // operator is prepared; a deeper split would have to reallocate it under
    // kernels already bound in the same trial batch
    if (k.split < 1 || k.split > OPEVO_MAX_SPLIT) {
        put_err(err, len, "split=%d out of range (1..%d)", k.split, OPEVO_MAX_SPLIT);
        return false;
    }
    if (!(k.acc == 1 || k.acc == 2 || k.acc == 4) || (k.bk / 16) % k.acc) {
        put_err(err, len, "acc=%d unsupported for BK=%d (1, 2 or 4 dividing BK/16)", k.acc, k.bk);
        return false;
    }
    if (!(k.cg == 1 || k.cg == 2) ||
        (k.cg == 2 && (k.bm < 256 || k.cluster != 1 || (family != 0 && family != 1) || b_resident(k, family)))) {
        put_err(err, len, "cta_group=%d needs BM=256 (or 512), no multicast cluster or resident weights", k.cg);
        return false;
    }
    if (!(k.bpu == 1 || k.bpu == 2 || k.bpu == 4) ||
        (k.bpu > 1 && (family != 0 || k.cg != 1 || k.cluster != 1 || k.bm != 128 || k.acc != 1 || k.split != 1 ||
                       (k.bk > 32 && k.bk % 64) || dsmem_split(k, family)))) {
        put_err(err, len, "bpu=%d needs a single-CTA 128-row GEMM tile, no multicast or DSMEM split", k.bpu);
        return false;
    }
    if (family == FAMILY_X3 && (k.cg != 1 || k.cluster != 1 || k.bpu > 1 || k.acc != 1 || k.b_res)) {
        put_err(err, len, "3xTF32: single-CTA tiles without multicast, bpu or acc");
        return false;
    }
    if (matoms_of(k) * k.bn * k.acc * std::max(1, k.bpu) > 512) {
        put_err(err, len, "accumulators %dx%d x%d exceed 512 TMEM columns", k.bm, k.bn, k.acc);
        return false;
    }
    if (!(k.cluster == 1 || k.cluster == 2 || k.cluster == 4 || k.cluster == 8) ||
        k.bm % (8 * k.cluster)) {
        put_err(err, len, "cluster=%d unsupported for BM=%d", k.cluster, k.bm);
        return false;
    }
    if (smem_bytes(k, family) > 232448) {
        put_err(err, len, "shared memory %zu B exceeds 227 KB", smem_bytes(k, family));
        return false;
    }
    if (family != 1 && k.line) {
        put_err(err, len, "padded lines are a conv tiling");
        return false;
    }
    if (family == 1) {
        const int bm_cta = bm_cta_of(k);               // tile rows held by one CTA
        if (k.cluster != 1) {
            put_err(err, len, "conv instances do not multicast");
            return false;
        }
        if (halo_kw(k, family)) {
            if (bm_cta % (16 * k.tile_h) || k.bk % 64 || k.split != 1) {
                put_err(err, len, "halo lines: %d rows must hold 16-row lines of %d rows, BK a multiple of 64, "
                        "no split", bm_cta, k.tile_h);
                return false;
            }
        } else if (k.line) {
            if (!(k.line == 16 || k.line == 32) || k.tile_w < 1 || k.tile_w > k.line || k.tile_h < 1 ||
                k.line * k.tile_h > bm_cta) {
                put_err(err, len, "padded lines: %d rows must hold at least one image of %d lines of %d rows "
                        "(16/32, >= TILE_W %d)", bm_cta, k.tile_h, k.line, k.tile_w);
                return false;
            }
        } else if (k.tile_h < 1 || k.tile_w < 1 || bm_cta % (k.tile_h * k.tile_w) || k.tile_w > 256 ||
                   k.tile_h > 256 || bm_cta / (k.tile_h * k.tile_w) > 256) {
            put_err(err, len, "conv tile %dx%d does not divide %d rows", k.tile_h, k.tile_w, bm_cta);
            return false;
        }
    }
    return true;
}

std::mutex g_fs_mu;

bool read_file(const std::string& path, std::vector<char>& out) {
    FILE* f = fopen(path.c_str(), "rb");
    if (!f) return false;
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    out.resize(n > 0 ? (size_t)n : 0);
    size_t got = n > 0 ? fread(out.data(), 1, (size_t)n, f) : 0;
    fclose(f);
    return n > 0 && got == (size_t)n;
}

void write_file_atomic(const std::string& path, const std::vector<char>& data) {
    char tmp[64];
    static std::atomic<unsigned> seq{0};
    snprintf(tmp, sizeof tmp, ".tmp.%d.%u", (int)getpid(), seq.fetch_add(1));
    std::string t = path + tmp;
    FILE* f = fopen(t.c_str(), "wb");
    if (!f) return;
    fwrite(data.data(), 1, data.size(), f);
    fclose(f);
    rename(t.c_str(), path.c_str());
}

void mkdirs(const std::string& dir) {
    std::string cur;
    for (size_t i = 0; i < dir.size(); ++i) {
        cur.push_back(dir[i]);
        if (dir[i] == '/' || i + 1 == dir.size()) mkdir(cur.c_str(), 0755);
    }
}

// NVRTC compile of one instance.  Returns status; cubin in `out`.
int nvrtc_build(int family, const Knobs& k, int batched, int out_f32, std::vector<char>& out,
                char* err, size_t len) {
    load_nvrtc();
    if (!g_rtc.ok) {
        put_err(err, len, "%s", g_rtc.why.c_str());
        return OPEVO_ERR_NO_NVRTC;
    }
    nvrtcProgram prog;
    const bool simt = family == 2;
    if (g_rtc.Create(&prog, simt ? opevo_sgemm_source : opevo_gemm_source,
                     simt ? "sgemm_simt.cuh" : "gemm_sm100.cuh", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        put_err(err, len, "nvrtcCreateProgram failed");
        return OPEVO_COMPILE_ERROR;
    }
    std::vector<std::string> opts;
    if (simt) {
        const Simt g = simt_of(k);
        opts = {"-arch=sm_100a", "-std=c++17", "-default-device",
                "-DOPEVO_N2=" + std::to_string(g.n2), "-DOPEVO_N3=" + std::to_string(g.n3),
                "-DOPEVO_N4=" + std::to_string(g.n4), "-DOPEVO_M2=" + std::to_string(g.m2),
                "-DOPEVO_M3=" + std::to_string(g.m3), "-DOPEVO_M4=" + std::to_string(g.m4),
                "-DOPEVO_K2=" + std::to_string(g.k2), "-DOPEVO_K3=" + std::to_string(g.k3)};
    } else opts = {
        "-arch=sm_100a", "-std=c++17", "-default-device",
        "-DOPEVO_BM=" + std::to_string(k.bm), "-DOPEVO_BN=" + std::to_string(k.bn),
        "-DOPEVO_BK=" + std::to_string(k.bk), "-DOPEVO_STAGES=" + std::to_string(k.stages),
        "-DOPEVO_BATCHED=" + std::to_string(batched), "-DOPEVO_OUT_F32=" + std::to_string(out_f32),
        "-DOPEVO_CLUSTER=" + std::to_string(k.cluster), "-DOPEVO_CONV=" + std::to_string(family == 1),
        "-DOPEVO_TILE_H=" + std::to_string(family == 1 ? k.tile_h : 1),
        "-DOPEVO_TILE_W=" + std::to_string(family == 1 ? k.tile_w : 1),
        "-DOPEVO_ACC=" + std::to_string(k.acc),
        "-DOPEVO_CTA_GROUP=" + std::to_string(k.cg),
        "-DOPEVO_SPLIT_CLUSTER=" + std::to_string(dsmem_split(k, family, batched) ? k.split : 0),
        "-DOPEVO_SPLIT_TMA=" + std::to_string(tma_split(k, family, batched)),
        "-DOPEVO_B_RES=" + std::to_string(b_resident(k, family) ? 1 : 0),
        "-DOPEVO_BPU=" + std::to_string(family == 0 ? std::max(1, k.bpu) : 1),
        "-DOPEVO_TF32X3=" + std::to_string(family == FAMILY_X3 ? 1 : 0),
        "-DOPEVO_HALO=" + std::to_string(halo_kw(k, family)),
        "-DOPEVO_LINE=" + std::to_string(family == 1 ? k.line : 0),
        "-DOPEVO_NARROW_EPI=" + std::to_string(narrow_epi(k, family, out_f32, batched) ? 1 : 0)};
    if (want_lineinfo()) opts.push_back("-lineinfo");
    {
        std::istringstream extra(instance_flags(family, k));
        std::string tok;
        while (extra >> tok) opts.push_back(tok);
    }
    std::vector<const char*> argv;
    for (auto& o : opts) argv.push_back(o.c_str());
    nvrtcResult r = g_rtc.Compile(prog, (int)argv.size(), argv.data());
    if (r != NVRTC_SUCCESS) {
        size_t n = 0;
        g_rtc.GetLogSize(prog, &n);
        std::string log(n, '\0');
        if (n) g_rtc.GetLog(prog, &log[0]);
        put_err(err, len, "NVRTC: %s: %s", g_rtc.ErrorString(r), log.c_str());
        g_rtc.Destroy(&prog);
        return OPEVO_COMPILE_ERROR;
    }
    size_t n = 0;
    g_rtc.GetCUBINSize(prog, &n);
    out.resize(n);
    g_rtc.GetCUBIN(prog, out.data());
    g_rtc.Destroy(&prog);
    return OPEVO_OK;
}

// Disk-cached compile: cache hit -> 2, compiled -> 0, failure -> status.
int get_cubin(int family, const Knobs& k, int batched, int out_f32, const std::string& cache_dir,
              std::vector<char>& cubin, double* compile_ms, int* hit, char* err, size_t len) {
    const std::string key = make_key(family, k, batched, out_f32);
    const std::string path = cache_dir.empty() ? "" : cache_dir + "/" + key + ".cubin";
    if (compile_ms) *compile_ms = 0.0;
    if (!path.empty() && read_file(path, cubin)) {
        if (hit) *hit = 2;
        return OPEVO_OK;
    }
    const double t0 = now_ms();
    int st = nvrtc_build(family, k, batched, out_f32, cubin, err, len);
    if (compile_ms) *compile_ms = now_ms() - t0;
    if (st != OPEVO_OK) return st;
    if (hit) *hit = 0;
    if (!path.empty()) {
        std::lock_guard<std::mutex> g(g_fs_mu);
        mkdirs(cache_dir);
        write_file_atomic(path, cubin);
    }
    return OPEVO_OK;
}

struct LoadedModule {
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
    int smem_set = 0;
};

}  // namespace

// Small persistent host pool: builds the timed graphs of a trial batch in
// parallel (capture + instantiate are host work) while the trial thread
// keeps the device busy with the batch's checks.
struct HostPool {
    std::vector<std::thread> threads;
    std::mutex mu;
    std::condition_variable cv, done_cv;
    std::vector<std::function<void(int)>> tasks;   // task(worker index)
    size_t next = 0, finished = 0;
    bool stop = false;

    void start(int n, CUcontext cu) {
        for (int w = 0; w < n; ++w)
            threads.emplace_back([this, w, cu] {
                g_cu.CtxSetCurrent(cu);
                std::unique_lock<std::mutex> lk(mu);
                while (true) {
                    cv.wait(lk, [this] { return stop || next < tasks.size(); });
                    if (stop) return;
                    auto fn = tasks[next++];
                    lk.unlock();
                    fn(w);
                    lk.lock();
                    if (++finished == tasks.size()) done_cv.notify_all();
                }
            });
    }
    void submit(std::vector<std::function<void(int)>> batch) {
        std::lock_guard<std::mutex> lk(mu);
        tasks = std::move(batch);
        next = finished = 0;
        cv.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        done_cv.wait(lk, [this] { return finished == tasks.size(); });
        tasks.clear();
        next = finished = 0;
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : threads) t.join();
    }
};

// ===================================================================== ctx
struct opevo_ctx {
    int device = 0;
    CUdevice dev = 0;
    CUcontext cu = nullptr;
    CUstream stream = nullptr;
    CUstream cap_stream = nullptr;      // graph capture of timed launches (overlaps the check)
    std::vector<CUstream> pool_streams; // one capture stream per graph-build worker
    std::unique_ptr<HostPool> pool;     // graph builds of a trial batch
    CUmodule util = nullptr;
    CUfunction k_fill_bf16 = nullptr, k_fill_f32 = nullptr, k_fill_u8 = nullptr, k_ref_gemm = nullptr,
               k_ref_gemm128 = nullptr, k_ref_gemm128x64 = nullptr,
               k_ref_conv = nullptr, k_ref_conv_tiled = nullptr, k_nchw2nhwc = nullptr, k_compare = nullptr, k_flush = nullptr,
               k_gate = nullptr, k_nchw2nhwc_pad = nullptr, k_nhwc_pad2nchw = nullptr;
    volatile uint32_t* gate_host = nullptr;   // mapped pinned flag opening the timing gate
    CUdeviceptr gate_dev = 0;
    uint32_t gate_seq = 0;
    CUdeviceptr flush_buf = 0;
    size_t flush_bytes = 0;
    CUdeviceptr cmp_buf = 0;
    int sm_count = 0, smem_optin = 0, cc_major = 0, cc_minor = 0;
    int smem_per_sm = 0, regs_per_sm = 0;
    // trial timing policy (opevo_ctx_set_timing)
    double budget_ms = 0.3;
    double loser_ratio = 0.0;
    int loser_reps = 5;
    std::string cache_dir;
    std::unordered_map<std::string, LoadedModule> modules;
    std::mutex modules_mu;              // modules may be preloaded from host pool threads
    bool poisoned = false;
};

struct opevo_op {
    opevo_ctx* ctx = nullptr;
    opevo_op_desc d{};
    int64_t rows = 0, cols = 0, depth = 0, batch = 1;   // GEMM view
    int64_t flop_depth = 0;                             // K of the operator (conv: unpadded Cin)
    int cpad = 0;                                       // conv: Cin in the kernel layout (16-aligned)
    size_t x_bytes = 0, w_bytes = 0;                    // conv: paper-layout operands
    CUdeviceptr a = 0, b = 0, c = 0, ref = 0;
    CUdeviceptr conv_x = 0, conv_w = 0;                 // paper layouts (NCHW / OIHW)
    CUdeviceptr ws = 0, counters = 0;
    size_t ws_bytes = 0, counter_bytes = 0;
    unsigned ws_gen = 0;                                // bumped when `ws` moves
    bool ref_stale = false;                             // operands uploaded since the reference
    float best_est_ms = 0.f;                            // fastest verified single launch (loser policy)
    size_t a_bytes = 0, b_bytes = 0, c_bytes = 0;
    int in_f32 = 0, out_f32 = 0;
    // Timed graphs by (knobs, repetitions).  Many configurations map to one
    // kernel instance (the thread-level factors have no tcgen05 counterpart),
    // so a generation often re-times an instance an earlier trial captured;
    // the graph's kernel arguments (tensor maps, pointers) are copied at
    // capture and stay valid until the split-K workspace is reallocated.
    std::unordered_map<std::string, CUgraphExec> graphs;
    // Instances verified on these operands (same cubin + launch plan: every
    // knob), with their verified launch's time.  Kernels are deterministic,
    // so a trial of an instance already verified here is re-timed but not
    // re-verified; uploading operands or recomputing the reference clears it.
    struct Verified { double rel_err; float est_ms; };
    std::unordered_map<std::string, Verified> verified;
};

namespace {
void drop_graphs(opevo_op* op) {
    for (auto& kv : op->graphs)
        if (kv.second) g_cu.GraphExecDestroy(kv.second);
    op->graphs.clear();
}

std::string graph_key(const Knobs& k, int reps) {
    char buf[160];
    snprintf(buf, sizeof buf, "%d_%d_%d_%d_%d_%d_%d_%d_%d_%d_%d_%d_%d_%d_r%d", k.bm, k.bn, k.bk, k.stages,
             k.split, k.cluster, k.tile_h, k.tile_w, k.acc, k.cg, k.grid_mode, k.b_res, k.bpu, k.line, reps);
    return buf;
}
}  // namespace

struct ConvGeomHost {
    int cin, ho, wo, kw, pad, taps_cchunks, stride;   // mirrors ConvGeom in gemm_sm100.cuh
};

// mirrors `Sched` in gemm_sm100.cuh
struct SchedHost {
    int row_tiles, col_groups, batches, split, head_tiles, tail_split, units;
};

struct opevo_kernel {
    opevo_op* op = nullptr;
    Knobs k{};
    int family = 0;
    CUfunction fn = nullptr;
    alignas(64) CUtensorMap tma_a;
    alignas(64) CUtensorMap tma_b;
    alignas(64) CUtensorMap tma_c;      // output, box = one 32-row epilogue chunk
    alignas(64) CUtensorMap tma_w{};    // TMA split-K partials {cols, rows, split} fp32 (else unused)
    unsigned ws_gen = 0;                // op->ws_gen tma_w was encoded against
    unsigned grid[3] = {1, 1, 1};
    size_t smem = 0;
    int k_per_split = 0;
    int kdepth = 0;                     // the kernel's `depth` argument (its K-loop extent)
    ConvGeomHost geom{};
    SchedHost sched{};
    std::atomic<int> launches{0};       // launches of this instance (all paths; graph
                                        // capture threads and the trial thread)
    unsigned block = 192;
    double flops = 0.0;
};

namespace {

int fail_cu(opevo_ctx* ctx, CUresult r, const char* what, char* err, size_t len) {
    put_err(err, len, "%s: %s (%d)", what, cu_str(r), (int)r);
    if (is_sticky(r)) {
        if (ctx) ctx->poisoned = true;
        return OPEVO_ERR_STICKY;
    }
    return OPEVO_ERR_CUDA;
}

#define CU_TRY(ctx, call, what)                                          \
    do {                                                                 \
        CUresult _r = (call);                                            \
        if (_r != CUDA_SUCCESS) return fail_cu((ctx), _r, (what), err, errlen); \
    } while (0)

unsigned grid_for(uint64_t n) {
    uint64_t g = (n + 255) / 256;
    return (unsigned)std::min<uint64_t>(std::max<uint64_t>(g, 1), 148 * 32);
}

int launch_simple(opevo_ctx* ctx, CUfunction f, unsigned grid, unsigned block, void** args, char* err,
                  size_t errlen) {
    CU_TRY(ctx, g_cu.LaunchKernel(f, grid, 1, 1, block, 1, 1, 0, ctx->stream, args, nullptr), "launch");
    return OPEVO_OK;
}

int fill(opevo_ctx* ctx, CUdeviceptr p, uint64_t n, uint64_t seed, int f32, char* err, size_t errlen) {
    void* args[] = {&p, &n, &seed};
    return launch_simple(ctx, f32 ? ctx->k_fill_f32 : ctx->k_fill_bf16, grid_for(n), 256, args, err,
                         errlen);
}

int compute_reference(opevo_op* op, char* err, size_t errlen) {
    opevo_ctx* ctx = op->ctx;
    if (op->d.kind == OPEVO_CONV2D) {
        const int32_t* c = op->d.conv;
        int N = c[0], C = c[1], H = c[2], W = c[3], K = c[4], KH = c[5], KW = c[6], S = c[7], P = c[8];
        int HO = (H + 2 * P - KH) / S + 1, WO = (W + 2 * P - KW) / S + 1;
        void* args[] = {&op->conv_x, &op->conv_w, &op->ref, &N, &C, &H, &W, &K, &KH, &KW, &S, &P, &HO, &WO};
        // tiled SIMT implicit GEMM (same fmaf chain per output as the
        // one-thread-per-output opevo_ref_conv, which remains as its check)
        const uint64_t pixels = (uint64_t)N * HO * WO;
        CU_TRY(ctx, g_cu.LaunchKernel(ctx->k_ref_conv_tiled, (unsigned)((pixels + 127) / 128),
                                      (unsigned)((K + 63) / 64), 1, 256, 1, 1, 0, ctx->stream, args, nullptr),
               "reference conv");
    } else {
        int rows = (int)op->rows, cols = (int)op->cols, depth = (int)op->depth, in_f32 = op->in_f32;
        void* args[] = {&op->a, &op->b, &op->ref, &rows, &cols, &depth, &in_f32};
        // large operands: the 128-row-tile references (bit-identical sums),
        // 128 x 64 tiles when 128 x 128 ones would not fill the SMs twice
        const bool big = rows >= 512 && cols >= 512;
        const bool narrow = big && (uint64_t)((rows + 127) / 128) * ((cols + 127) / 128) * op->batch <
                                       (uint64_t)ctx->sm_count * 2;
        const unsigned tr = big ? 128u : 64u, tc = big && !narrow ? 128u : 64u;
        CUfunction fn = !big ? ctx->k_ref_gemm : narrow ? ctx->k_ref_gemm128x64 : ctx->k_ref_gemm128;
        CU_TRY(ctx, g_cu.LaunchKernel(fn, (unsigned)((cols + tc - 1) / tc),
                                      (unsigned)((rows + tr - 1) / tr), (unsigned)op->batch, 256, 1, 1, 0,
                                      ctx->stream, args, nullptr),
               "reference gemm");
    }
    CU_TRY(ctx, g_cu.StreamSynchronize(ctx->stream), "reference sync");
    return OPEVO_OK;
}

// Before any check: a reference made stale by opevo_op_upload is recomputed
// from the uploaded operands.
int fresh_reference(opevo_op* op, char* err, size_t errlen) {
    if (!op->ref_stale) return OPEVO_OK;
    op->ref_stale = false;
    op->verified.clear();
    return compute_reference(op, err, errlen);
}

int ensure_ws(opevo_op* op, size_t ws_need, size_t cnt_need, char* err, size_t errlen) {
    opevo_ctx* ctx = op->ctx;
    if (ws_need > op->ws_bytes || cnt_need > op->counter_bytes) drop_graphs(op);   // captured pointers go stale
    if (ws_need > op->ws_bytes) {
        ++op->ws_gen;                                   // bound TMA split maps re-encode
        if (op->ws) g_cu.MemFree(op->ws);
        op->ws = 0;
        op->ws_bytes = 0;
        CU_TRY(ctx, g_cu.MemAlloc(&op->ws, ws_need), "alloc split-K workspace");
        op->ws_bytes = ws_need;
    }
    if (cnt_need > op->counter_bytes) {
        if (op->counters) g_cu.MemFree(op->counters);
        op->counters = 0;
        op->counter_bytes = 0;
        CU_TRY(ctx, g_cu.MemAlloc(&op->counters, cnt_need), "alloc tile counters");
        CU_TRY(ctx, g_cu.MemsetD8(op->counters, 0, cnt_need), "zero tile counters");
        op->counter_bytes = cnt_need;
    }
    return OPEVO_OK;
}

CUtensorMapSwizzle swz_enum(int bytes) {
    return bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                        : bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
}

int encode_map(CUtensorMap* map, CUdeviceptr base, int rank, const uint64_t* dims, const uint64_t* strides_b,
               const uint32_t* box, int swz, char* err, size_t errlen, int f32 = 0,
               const uint32_t* elem_strides = nullptr) {
    uint32_t es[5] = {1, 1, 1, 1, 1};
    if (elem_strides)
        for (int i = 0; i < rank; ++i) es[i] = elem_strides[i];
    CUresult r = g_cu.TensorMapEncodeTiled(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                           (cuuint32_t)rank,
                                           (void*)base, (const cuuint64_t*)dims,
                                           (const cuuint64_t*)strides_b, (const cuuint32_t*)box,
                                           (const cuuint32_t*)es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           swz_enum(swz), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        put_err(err, errlen, "cuTensorMapEncodeTiled: %s", cu_str(r));
        return OPEVO_INVALID_CONFIG;
    }
    return OPEVO_OK;
}

// TMA split-K partials {cols, rows, split} fp32 in op->ws.  Recorded against
// op->ws_gen, so a kernel bound before the workspace moved re-encodes it at
// its next launch instead of storing into freed memory.
int encode_split_map(opevo_kernel* kr, int tsplit, char* err, size_t errlen) {
    opevo_op* op = kr->op;
    uint64_t wd[3] = {(uint64_t)op->cols, (uint64_t)op->rows, (uint64_t)tsplit};
    uint64_t wstr[2] = {(uint64_t)op->cols * 4, (uint64_t)op->cols * op->rows * 4};
    uint32_t wb[3] = {32, 32, 1};
    kr->ws_gen = op->ws_gen;
    return encode_map(&kr->tma_w, op->ws, 3, wd, wstr, wb, 128, err, errlen, 1);
}

int launch_kernel(opevo_kernel* kr, char* err, size_t errlen, CUstream on = nullptr) {
    opevo_op* op = kr->op;
    opevo_ctx* ctx = op->ctx;
    CUstream strm = on ? on : ctx->stream;
    if (kr->family == 2) {
        int rows = (int)op->rows, cols = (int)op->cols, depth = (int)op->depth;
        void* args[] = {&op->a, &op->b, &op->c, &rows, &cols, &depth};
        CUlaunchConfig cfg{};
        cfg.gridDimX = kr->grid[0];
        cfg.gridDimY = kr->grid[1];
        cfg.gridDimZ = kr->grid[2];
        cfg.blockDimX = kr->block;
        cfg.blockDimY = cfg.blockDimZ = 1;
        cfg.sharedMemBytes = (unsigned)kr->smem;
        cfg.hStream = strm;
        CUlaunchAttribute attr[1];
        if (want_pdl()) {
            attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
            attr[0].value.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
        }
        CUresult r = g_cu.LaunchKernelEx(&cfg, kr->fn, args, nullptr);
        if (strm == ctx->stream) ++kr->launches;   // captured launches count when the graph runs
        if (r != CUDA_SUCCESS) {
            int st = fail_cu(ctx, r, "kernel launch", err, errlen);
            return st == OPEVO_ERR_STICKY ? st : OPEVO_LAUNCH_ERROR;
        }
        return OPEVO_OK;
    }
    const int batched = op->d.kind == OPEVO_BATCHMATMUL ? 1 : 0;
    if (kr->ws_gen != op->ws_gen) {
        if (const int ts = tma_split(kr->k, kr->family, batched)) {
            const int est = encode_split_map(kr, ts, err, errlen);
            if (est) return est;
        }
        kr->ws_gen = op->ws_gen;
    }
    int rows = (int)op->rows;
    int cols = (int)op->cols;
    int depth = kr->kdepth;                        // K-loop extent (bf16 units for 3xTF32)
    void* cptr = (void*)op->c;
    float* ws = (float*)op->ws;
    unsigned* cnt = (unsigned*)op->counters;
    void* args[] = {&kr->tma_a, &kr->tma_b, &kr->tma_c, &kr->tma_w, &cptr, &ws, &cnt, &rows, &cols, &depth, &kr->sched,
                    &kr->geom};
    CUlaunchConfig cfg{};
    cfg.gridDimX = kr->grid[0];
    cfg.gridDimY = kr->grid[1];
    cfg.gridDimZ = kr->grid[2];
    cfg.blockDimX = 192;
    cfg.blockDimY = 1;
    cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)kr->smem;
    cfg.hStream = strm;
    CUlaunchAttribute attr[2];
    unsigned na = 0;
    const unsigned clx = (unsigned)(kr->k.cluster * kr->k.cg *
                                    (dsmem_split(kr->k, kr->family, batched) ? kr->k.split : 1));
    if (clx > 1) {
        attr[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
        attr[na].value.clusterDim.x = clx;
        attr[na].value.clusterDim.y = 1;
        attr[na].value.clusterDim.z = 1;
        ++na;
    }
    if (want_pdl()) {
        // programmatic dependent launch: the kernel calls griddepcontrol.wait
        // before touching global memory, so its prologue may overlap the
        // previous kernel in the stream
        attr[na].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
        attr[na].value.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
    CUresult r = g_cu.LaunchKernelEx(&cfg, kr->fn, args, nullptr);
    if (strm == ctx->stream) ++kr->launches;       // captured launches count when the graph runs
    if (r != CUDA_SUCCESS) {
        int st = fail_cu(ctx, r, "kernel launch", err, errlen);
        return st == OPEVO_ERR_STICKY ? st : OPEVO_LAUNCH_ERROR;
    }
    return OPEVO_OK;
}

int sync_checked(opevo_ctx* ctx, const char* what, char* err, size_t errlen) {
    CUresult r = g_cu.StreamSynchronize(ctx->stream);
    if (r != CUDA_SUCCESS) {
        int st = fail_cu(ctx, r, what, err, errlen);
        return st == OPEVO_ERR_STICKY ? st : OPEVO_LAUNCH_ERROR;
    }
    return OPEVO_OK;
}

// Module for an instance: per-context memory cache -> disk cache -> NVRTC.
int get_function(opevo_ctx* ctx, int family, const Knobs& k, int batched, int out_f32, const char* name,
                 size_t smem, CUfunction* fn, double* compile_ms, int* hit, char* err, size_t errlen) {
    const std::string key = make_key(family, k, batched, out_f32);
    *compile_ms = 0.0;
    *hit = 1;
    std::unique_lock<std::mutex> lock(ctx->modules_mu);
    auto it = ctx->modules.find(key);
    if (it == ctx->modules.end()) {
        // compile / read and load outside the lock (preload threads run this too)
        lock.unlock();
        std::vector<char> cubin;
        int st = get_cubin(family, k, batched, out_f32, ctx->cache_dir, cubin, compile_ms, hit, err, errlen);
        if (st) return st;
        LoadedModule lm;
        CUresult r = g_cu.ModuleLoadData(&lm.mod, cubin.data());
        if (r == CUDA_SUCCESS) r = g_cu.ModuleGetFunction(&lm.fn, lm.mod, name);
        // Under lazy module loading (the CUDA 12 default) the code would reach
        // the device at its first launch or graph instantiation -- on the
        // trial's critical path, holding the driver lock for milliseconds.
        // Load it here, on the preload thread.
        if (r == CUDA_SUCCESS) r = g_cu.FuncLoad(lm.fn);
        if (r != CUDA_SUCCESS) {
            st = fail_cu(ctx, r, "load module", err, errlen);
            return st == OPEVO_ERR_STICKY ? st : OPEVO_LAUNCH_ERROR;
        }
        lock.lock();
        auto ins = ctx->modules.emplace(key, lm);
        if (!ins.second) g_cu.ModuleUnload(lm.mod);      // another thread won the race
        it = ins.first;
    }
    LoadedModule& lm = it->second;
    if (smem > 0 && lm.smem_set < (int)smem) {
        CUresult r = g_cu.FuncSetAttribute(lm.fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
        if (r != CUDA_SUCCESS) {
            put_err(err, errlen, "set smem %zu: %s", smem, cu_str(r));
            return OPEVO_INVALID_CONFIG;
        }
        lm.smem_set = (int)smem;
    }
    *fn = lm.fn;
    return OPEVO_OK;
}

// fp32 SIMT family (paper TVM dense schedule): plain pointers, 3-D grid.
int simt_kernel_get(opevo_ctx* ctx, opevo_op* op, const Knobs& k, opevo_kernel** out,
                    opevo_trial_result* info, double t0, char* err, size_t errlen) {
    const Simt g = simt_of(k);
    if (op->rows % g.bm() || op->cols % g.bn() || op->depth % g.ks()) {
        put_err(err, errlen, "SIMT tile %dx%d (k chunk %d) does not divide %lldx%lldx%lld", g.bm(), g.bn(),
                g.ks(), (long long)op->rows, (long long)op->cols, (long long)op->depth);
        return OPEVO_INVALID_CONFIG;
    }
    if ((int)g.smem() > ctx->smem_optin) {
        put_err(err, errlen, "shared memory %zu B exceeds the device limit", g.smem());
        return OPEVO_INVALID_CONFIG;
    }
    opevo_kernel* kr = new opevo_kernel();
    kr->op = op;
    kr->k = k;
    kr->family = 2;
    kr->smem = g.smem();
    kr->block = (unsigned)g.threads();
    kr->grid[0] = (unsigned)(op->cols / g.bn());
    kr->grid[1] = (unsigned)(op->rows / g.bm());
    kr->grid[2] = (unsigned)op->batch;
    kr->flops = 2.0 * (double)op->batch * (double)op->rows * (double)op->cols * (double)op->flop_depth;
    double compile_ms = 0.0;
    int hit = 1;
    int st = get_function(ctx, 2, k, op->d.kind == OPEVO_BATCHMATMUL, 1, "opevo_sgemm", kr->smem, &kr->fn,
                          &compile_ms, &hit, err, errlen);
    if (st) {
        delete kr;
        return st;
    }
    if (info) {
        info->compile_ms = compile_ms;
        info->cache_hit = hit;
        info->load_ms = now_ms() - t0 - compile_ms;
        info->grid_ctas = (int32_t)(kr->grid[0] * kr->grid[1] * kr->grid[2]);
        info->smem_bytes = (int32_t)kr->smem;
    }
    *out = kr;
    return OPEVO_OK;
}

}  // namespace

// ================================================================= exports
extern "C" {

int opevo_abi_version(void) { return OPEVO_ABI_VERSION; }

int opevo_kernel_key(int family, const int32_t* knobs, int nknobs, int batched, int out_f32, char* key,
                     size_t keylen) {
    if (!knobs || !key) return OPEVO_ERR_ARG;
    std::string s = make_key(family, lib_knobs(family, knobs, nknobs), batched, out_f32);
    snprintf(key, keylen, "%s", s.c_str());
    return OPEVO_OK;
}

int opevo_compile(int family, const int32_t* knobs, int nknobs, int batched, int out_f32,
                  const char* cache_dir, double* compile_ms, char* err, size_t errlen) {
    if (!knobs) return OPEVO_ERR_ARG;
    Knobs k = lib_knobs(family, knobs, nknobs);
    if (!knobs_compilable(family, k, err, errlen)) return OPEVO_INVALID_CONFIG;
    std::vector<char> cubin;
    int hit = 0;
    return get_cubin(family, k, batched, out_f32, cache_dir ? cache_dir : "", cubin, compile_ms, &hit,
                     err, errlen);
}

int opevo_ctx_create(int device, const char* cache_dir, opevo_ctx** out, char* err, size_t errlen) {
    if (!out) return OPEVO_ERR_ARG;
    *out = nullptr;
    load_driver();
    if (!g_cu.ok) {
        put_err(err, errlen, "%s", g_cu.why.c_str());
        return OPEVO_ERR_NO_DEVICE;
    }
    opevo_ctx* ctx = new opevo_ctx();
    ctx->device = device;
    if (const char* b = getenv("OPEVO_TIME_BUDGET_MS")) ctx->budget_ms = atof(b);
    ctx->cache_dir = cache_dir ? cache_dir : "";
    CUresult r = g_cu.DeviceGet(&ctx->dev, device);
    if (r != CUDA_SUCCESS) {
        put_err(err, errlen, "cuDeviceGet(%d): %s", device, cu_str(r));
        delete ctx;
        return OPEVO_ERR_NO_DEVICE;
    }
    if ((r = g_cu.PrimaryCtxRetain(&ctx->cu, ctx->dev)) != CUDA_SUCCESS ||
        (r = g_cu.CtxSetCurrent(ctx->cu)) != CUDA_SUCCESS) {
        put_err(err, errlen, "primary context: %s", cu_str(r));
        delete ctx;
        return OPEVO_ERR_NO_DEVICE;
    }
    g_cu.DeviceGetAttribute(&ctx->sm_count, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, ctx->dev);
    g_cu.DeviceGetAttribute(&ctx->smem_optin, CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_BLOCK_OPTIN, ctx->dev);
    g_cu.DeviceGetAttribute(&ctx->smem_per_sm, CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_MULTIPROCESSOR, ctx->dev);
    g_cu.DeviceGetAttribute(&ctx->regs_per_sm, CU_DEVICE_ATTRIBUTE_MAX_REGISTERS_PER_MULTIPROCESSOR, ctx->dev);
    g_cu.DeviceGetAttribute(&ctx->cc_major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, ctx->dev);
    g_cu.DeviceGetAttribute(&ctx->cc_minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, ctx->dev);
    if (ctx->cc_major != 10) {
        put_err(err, errlen, "device %d is sm_%d%d; this build targets sm_100a only", device,
                ctx->cc_major, ctx->cc_minor);
        g_cu.PrimaryCtxRelease(ctx->dev);
        delete ctx;
        return OPEVO_ERR_NO_DEVICE;
    }
    int st = OPEVO_OK;
    auto bail = [&](CUresult rr, const char* what) {
        st = fail_cu(ctx, rr, what, err, errlen);
    };
    if ((r = g_cu.StreamCreate(&ctx->stream, CU_STREAM_NON_BLOCKING)) != CUDA_SUCCESS) bail(r, "stream");
    else if ((r = g_cu.StreamCreate(&ctx->cap_stream, CU_STREAM_NON_BLOCKING)) != CUDA_SUCCESS)
        bail(r, "capture stream");
    else if ((r = g_cu.ModuleLoadData(&ctx->util, opevo_util_cubin)) != CUDA_SUCCESS) bail(r, "load util cubin");
    else if ((r = g_cu.MemAlloc(&ctx->cmp_buf, 16 * OPEVO_MAX_BATCH)) != CUDA_SUCCESS) bail(r, "alloc");
    if (st == OPEVO_OK) {
        struct { CUfunction* f; const char* n; } fns[] = {
            {&ctx->k_fill_bf16, "opevo_fill_bf16"}, {&ctx->k_fill_f32, "opevo_fill_f32"},
            {&ctx->k_fill_u8, "opevo_fill_u8"},     {&ctx->k_ref_gemm, "opevo_ref_gemm"},
            {&ctx->k_ref_gemm128, "opevo_ref_gemm128"},   {&ctx->k_ref_gemm128x64, "opevo_ref_gemm128x64"},
            {&ctx->k_ref_conv, "opevo_ref_conv"},   {&ctx->k_ref_conv_tiled, "opevo_ref_conv_tiled"},   {&ctx->k_nchw2nhwc, "opevo_nchw_to_nhwc"},
            {&ctx->k_compare, "opevo_compare"},     {&ctx->k_flush, "opevo_flush"},
            {&ctx->k_gate, "opevo_gate"},           {&ctx->k_nchw2nhwc_pad, "opevo_nchw_to_nhwc_pad"},
            {&ctx->k_nhwc_pad2nchw, "opevo_nhwc_pad_to_nchw"}};
        for (auto& f : fns) {
            if ((r = g_cu.ModuleGetFunction(f.f, ctx->util, f.n)) != CUDA_SUCCESS) {
                bail(r, f.n);
                break;
            }
        }
    }
    if (st == OPEVO_OK) {
        void* hp = nullptr;
        if ((r = g_cu.MemHostAlloc(&hp, 64, CU_MEMHOSTALLOC_DEVICEMAP | CU_MEMHOSTALLOC_PORTABLE)) != CUDA_SUCCESS)
            bail(r, "alloc gate flag");
        else if ((r = g_cu.MemHostGetDevicePointer(&ctx->gate_dev, hp, 0)) != CUDA_SUCCESS)
            bail(r, "map gate flag");
        if (hp) {
            ctx->gate_host = static_cast<volatile uint32_t*>(hp);
            *ctx->gate_host = 0;
        }
    }
    if (st != OPEVO_OK) {
        opevo_ctx_destroy(ctx);
        return st;
    }
    *out = ctx;
    return OPEVO_OK;
}

void opevo_ctx_destroy(opevo_ctx* ctx) {
    if (!ctx) return;
    if (g_cu.ok && !ctx->poisoned) {
        g_cu.CtxSetCurrent(ctx->cu);
        for (auto& kv : ctx->modules)
            if (kv.second.mod) g_cu.ModuleUnload(kv.second.mod);
        if (ctx->util) g_cu.ModuleUnload(ctx->util);
        if (ctx->flush_buf) g_cu.MemFree(ctx->flush_buf);
        if (ctx->cmp_buf) g_cu.MemFree(ctx->cmp_buf);
        if (ctx->gate_host) g_cu.MemFreeHost((void*)ctx->gate_host);
        if (ctx->stream) g_cu.StreamDestroy(ctx->stream);
        if (ctx->cap_stream) g_cu.StreamDestroy(ctx->cap_stream);
        ctx->pool.reset();
        for (CUstream st : ctx->pool_streams) g_cu.StreamDestroy(st);
        g_cu.PrimaryCtxRelease(ctx->dev);
    }
    delete ctx;
}

int opevo_ctx_info(opevo_ctx* ctx, int* sm_count, int* max_smem_optin, int* cc_major, int* cc_minor) {
    if (!ctx) return OPEVO_ERR_ARG;
    if (sm_count) *sm_count = ctx->sm_count;
    if (max_smem_optin) *max_smem_optin = ctx->smem_optin;
    if (cc_major) *cc_major = ctx->cc_major;
    if (cc_minor) *cc_minor = ctx->cc_minor;
    return OPEVO_OK;
}

void opevo_op_destroy(opevo_op* op) {
    if (!op) return;
    if (g_cu.ok && op->ctx && !op->ctx->poisoned) {
        g_cu.CtxSetCurrent(op->ctx->cu);
        drop_graphs(op);
        CUdeviceptr ps[] = {op->a, op->b, op->c, op->ref, op->conv_x, op->conv_w, op->ws, op->counters};
        for (CUdeviceptr p : ps)
            if (p) g_cu.MemFree(p);
    }
    delete op;
}

int opevo_op_prepare(opevo_ctx* ctx, const opevo_op_desc* desc, opevo_op** out, char* err, size_t errlen) {
    if (!ctx || !desc || !out) return OPEVO_ERR_ARG;
    if (ctx->poisoned) {
        put_err(err, errlen, "context poisoned by an earlier fault");
        return OPEVO_ERR_STICKY;
    }
    *out = nullptr;
    g_cu.CtxSetCurrent(ctx->cu);
    opevo_op* op = new opevo_op();
    op->ctx = ctx;
    op->d = *desc;
    if (desc->dtype == OPEVO_F32_TF32X3 && desc->kind == OPEVO_CONV2D) {
        put_err(err, errlen, "3xTF32 is served for MatMul / BatchMatMul");
        delete op;
        return OPEVO_ERR_ARG;
    }
    op->in_f32 = op->out_f32 = (desc->dtype == OPEVO_F32 || desc->dtype == OPEVO_F32_TF32X3) ? 1 : 0;
    const size_t esz = op->in_f32 ? 4 : 2;
    int st = OPEVO_OK;
    auto alloc = [&](CUdeviceptr* p, size_t bytes, const char* what) -> bool {
        CUresult r = g_cu.MemAlloc(p, std::max<size_t>(bytes, 16));
        if (r != CUDA_SUCCESS) {
            st = fail_cu(ctx, r, what, err, errlen);
            return false;
        }
        return true;
    };
    if (desc->kind == OPEVO_MATMUL || desc->kind == OPEVO_BATCHMATMUL) {
        op->batch = desc->kind == OPEVO_MATMUL ? 1 : desc->batch;
        op->rows = desc->rows;
        op->cols = desc->cols;
        op->depth = desc->depth;
        if (op->batch < 1 || op->rows < 1 || op->cols < 1 || op->depth < 1) {
            put_err(err, errlen, "non-positive operator dimension");
            delete op;
            return OPEVO_ERR_ARG;
        }
        op->flop_depth = op->depth;
        op->a_bytes = (size_t)op->batch * op->rows * op->depth * esz;
        op->b_bytes = (size_t)op->batch * op->cols * op->depth * esz;
        op->c_bytes = (size_t)op->batch * op->rows * op->cols * (op->out_f32 ? 4 : 2);
        if (alloc(&op->a, op->a_bytes, "alloc A") && alloc(&op->b, op->b_bytes, "alloc B") &&
            alloc(&op->c, op->c_bytes, "alloc C") &&
            alloc(&op->ref, (size_t)op->batch * op->rows * op->cols * 4, "alloc reference")) {
            st = fill(ctx, op->a, op->a_bytes / esz, desc->seed, op->in_f32, err, errlen);
            if (!st) st = fill(ctx, op->b, op->b_bytes / esz, desc->seed + 1, op->in_f32, err, errlen);
        }
    } else if (desc->kind == OPEVO_CONV2D) {
        const int32_t* c = desc->conv;
        int N = c[0], C = c[1], H = c[2], W = c[3], K = c[4], KH = c[5], KW = c[6], S = c[7], P = c[8];
        if (desc->dtype != OPEVO_BF16 || N < 1 || C < 1 || H < 1 || W < 1 || K < 1 || KH < 1 || KW < 1 ||
            S < 1 || P < 0) {
            put_err(err, errlen, "invalid conv2d descriptor");
            delete op;
            return OPEVO_ERR_ARG;
        }
        int HO = (H + 2 * P - KH) / S + 1, WO = (W + 2 * P - KW) / S + 1;
        if (HO < 1 || WO < 1) {
            put_err(err, errlen, "conv2d output is empty");
            delete op;
            return OPEVO_ERR_ARG;
        }
        // kernel layouts: X NHWC and W [Cout][Kh][Kw][Cin] with Cin padded
        // with zeros to a multiple of 16 (one 32-byte UMMA K step; a TMA
        // row must be >= 16 bytes), e.g. AlexNet conv1's Cin = 3 -> 16
        int CP = (C + 15) / 16 * 16;
        op->cpad = CP;
        op->batch = 1;
        op->rows = (int64_t)N * HO * WO;
        op->cols = K;
        op->depth = (int64_t)KH * KW * CP;
        op->flop_depth = (int64_t)KH * KW * C;
        op->x_bytes = (size_t)N * C * H * W * 2;
        op->w_bytes = (size_t)K * C * KH * KW * 2;
        op->a_bytes = (size_t)N * H * W * CP * 2;
        op->b_bytes = (size_t)K * KH * KW * CP * 2;
        op->c_bytes = (size_t)op->rows * op->cols * 2;
        if (alloc(&op->conv_x, op->x_bytes, "alloc X") && alloc(&op->conv_w, op->w_bytes, "alloc W") &&
            alloc(&op->a, op->a_bytes, "alloc X nhwc") && alloc(&op->b, op->b_bytes, "alloc W ohwi") &&
            alloc(&op->c, op->c_bytes, "alloc C") && alloc(&op->ref, (size_t)op->rows * op->cols * 4, "alloc ref")) {
            st = fill(ctx, op->conv_x, op->x_bytes / 2, desc->seed, 0, err, errlen);
            if (!st) st = fill(ctx, op->conv_w, op->w_bytes / 2, desc->seed + 1, 0, err, errlen);
            if (!st) {
                // NCHW -> NHWC (channels padded with zeros to CP)
                uint64_t n1 = op->a_bytes / 2;
                void* a1[] = {&op->conv_x, &op->a, &N, &C, &H, &W, &CP};
                st = launch_simple(ctx, ctx->k_nchw2nhwc_pad, grid_for(n1), 256, a1, err, errlen);
            }
            if (!st) {
                // OIHW viewed as [O][I][KH][KW] -> [O][KH][KW][I padded]
                uint64_t n2 = op->b_bytes / 2;
                void* a2[] = {&op->conv_w, &op->b, &K, &C, &KH, &KW, &CP};
                st = launch_simple(ctx, ctx->k_nchw2nhwc_pad, grid_for(n2), 256, a2, err, errlen);
            }
        }
    } else {
        put_err(err, errlen, "unknown operator kind %d", desc->kind);
        delete op;
        return OPEVO_ERR_ARG;
    }
    if (!st) st = compute_reference(op, err, errlen);
    if (!st) {
        // split-K workspace for OPEVO_MAX_SPLIT slices and tile counters, up front:
        // growing them during a search reallocates (and drops the timed
        // graphs that captured the old pointers) on the trial's critical path
        const size_t slice = (size_t)op->batch * op->rows * op->cols * 4;
        const size_t tiles = (size_t)op->batch * ((op->rows + 127) / 128) * ((op->cols + 15) / 16);
        st = ensure_ws(op, slice * OPEVO_MAX_SPLIT, tiles * 16 * 4, err, errlen);
    }
    if (st) {
        opevo_op_destroy(op);
        return st;
    }
    *out = op;
    return OPEVO_OK;
}

int opevo_op_sizes(const opevo_op* op, size_t* a_bytes, size_t* b_bytes, size_t* c_bytes) {
    if (!op) return OPEVO_ERR_ARG;
    if (a_bytes) *a_bytes = op->a_bytes;
    if (b_bytes) *b_bytes = op->b_bytes;
    if (c_bytes) *c_bytes = op->c_bytes;
    return OPEVO_OK;
}

int opevo_op_upload(opevo_op* op, const void* a_host, const void* b_host, char* err, size_t errlen) {
    if (!op) return OPEVO_ERR_ARG;
    opevo_ctx* ctx = op->ctx;
    g_cu.CtxSetCurrent(ctx->cu);
    if (a_host) CU_TRY(ctx, g_cu.MemcpyHtoDAsync(op->a, a_host, op->a_bytes, ctx->stream), "upload A");
    if (b_host) CU_TRY(ctx, g_cu.MemcpyHtoDAsync(op->b, b_host, op->b_bytes, ctx->stream), "upload B");
    if (op->d.kind == OPEVO_CONV2D && (a_host || b_host)) {
        // the reference convolves the paper's layouts: NHWC (channels padded
        // to CP) -> NCHW, and [O][KH][KW][I padded] -> OIHW
        const int32_t* c = op->d.conv;
        int N = c[0], C = c[1], H = c[2], W = c[3], K = c[4], KH = c[5], KW = c[6], CP = op->cpad;
        int st = OPEVO_OK;
        if (a_host) {
            void* a1[] = {&op->a, &op->conv_x, &N, &C, &H, &W, &CP};
            st = launch_simple(ctx, ctx->k_nhwc_pad2nchw, grid_for(op->x_bytes / 2), 256, a1, err, errlen);
        }
        if (!st && b_host) {
            void* a2[] = {&op->b, &op->conv_w, &K, &C, &KH, &KW, &CP};
            st = launch_simple(ctx, ctx->k_nhwc_pad2nchw, grid_for(op->w_bytes / 2), 256, a2, err, errlen);
        }
        if (st) return st;
    }
    if (a_host || b_host) {
        op->verified.clear();             // new operands: every instance is verified again
        op->ref_stale = true;             // and against a reference recomputed from them
    }
    return OPEVO_OK;
}

int opevo_op_download(opevo_op* op, void* c_host, size_t bytes, char* err, size_t errlen) {
    if (!op || !c_host) return OPEVO_ERR_ARG;
    opevo_ctx* ctx = op->ctx;
    g_cu.CtxSetCurrent(ctx->cu);
    CU_TRY(ctx, g_cu.MemcpyDtoHAsync(c_host, op->c, std::min(bytes, op->c_bytes), ctx->stream), "download C");
    CU_TRY(ctx, g_cu.StreamSynchronize(ctx->stream), "download sync");
    return OPEVO_OK;
}

int opevo_op_read_inputs(opevo_op* op, void* a_host, void* b_host, char* err, size_t errlen) {
    if (!op) return OPEVO_ERR_ARG;
    opevo_ctx* ctx = op->ctx;
    g_cu.CtxSetCurrent(ctx->cu);
    CU_TRY(ctx, g_cu.StreamSynchronize(ctx->stream), "sync");
    if (a_host) CU_TRY(ctx, g_cu.MemcpyDtoH(a_host, op->a, op->a_bytes), "read A");
    if (b_host) CU_TRY(ctx, g_cu.MemcpyDtoH(b_host, op->b, op->b_bytes), "read B");
    return OPEVO_OK;
}

int opevo_op_reference(opevo_op* op, float* host, size_t count, char* err, size_t errlen) {
    if (!op || !host) return OPEVO_ERR_ARG;
    opevo_ctx* ctx = op->ctx;
    g_cu.CtxSetCurrent(ctx->cu);
    size_t n = std::min<size_t>(count, (size_t)op->batch * op->rows * op->cols);
    if (int st = fresh_reference(op, err, errlen)) return st;
    CU_TRY(ctx, g_cu.StreamSynchronize(ctx->stream), "sync");
    CU_TRY(ctx, g_cu.MemcpyDtoH(host, op->ref, n * 4), "download reference");
    return OPEVO_OK;
}

int opevo_op_refresh_reference(opevo_op* op, char* err, size_t errlen) {
    if (!op) return OPEVO_ERR_ARG;
    g_cu.CtxSetCurrent(op->ctx->cu);
    op->verified.clear();
    op->ref_stale = false;
    return compute_reference(op, err, errlen);
}

int opevo_kernel_get(opevo_ctx* ctx, opevo_op* op, const int32_t* knobs, int nknobs, opevo_kernel** out,
                     opevo_trial_result* info, char* err, size_t errlen) {
    if (!ctx || !op || !knobs || !out) return OPEVO_ERR_ARG;
    *out = nullptr;
    if (ctx->poisoned) {
        put_err(err, errlen, "context poisoned by an earlier fault");
        return OPEVO_ERR_STICKY;
    }
    g_cu.CtxSetCurrent(ctx->cu);
    const double t0 = now_ms();
    // fp32 operands: the SIMT family (OPEVO_F32) or 3xTF32 on tcgen05 (OPEVO_F32_TF32X3)
    const int family = family_of(op->d);
    Knobs k = lib_knobs(family, knobs, nknobs);
    // K as the kernel sees it (bf16 units: doubled for the 3xTF32 family)
    const int64_t depth = op->depth * (family == FAMILY_X3 ? 2 : 1);
    const int batched = op->d.kind == OPEVO_BATCHMATMUL ? 1 : 0;
    if (!knobs_compilable(family, k, err, errlen)) return OPEVO_INVALID_CONFIG;
    if (family == 2) return simt_kernel_get(ctx, op, k, out, info, t0, err, errlen);
    if ((int)smem_bytes(k, family, op->out_f32, batched) > ctx->smem_optin) {
        put_err(err, errlen, "shared memory %zu B exceeds the device limit %d", smem_bytes(k, family, op->out_f32, batched),
                ctx->smem_optin);
        return OPEVO_INVALID_CONFIG;
    }
    // operator-dependent feasibility (divisibility: no tail handling by design)
    // (halo-line conv tiles hold 16 * lines rows for TILE_W * lines pixels;
    // the conv branch checks their tiling)
    if ((op->rows % k.bm && family != 1) || op->cols % k.bn) {
        put_err(err, errlen, "tile %dx%d does not divide %lldx%lld", k.bm, k.bn, (long long)op->rows,
                (long long)op->cols);
        return OPEVO_INVALID_CONFIG;
    }
    if (k.split < 1 || depth % ((int64_t)k.split * k.bk)) {
        put_err(err, errlen, "split %d x BK %d does not divide K=%lld", k.split, k.bk, (long long)depth);
        return OPEVO_INVALID_CONFIG;
    }
    const int64_t col_tiles = op->cols / k.bn, row_tiles = op->rows / k.bm;
    if (col_tiles % k.cluster) {
        put_err(err, errlen, "cluster %d does not divide %lld column tiles", k.cluster, (long long)col_tiles);
        return OPEVO_INVALID_CONFIG;
    }
    opevo_kernel* kr = new opevo_kernel();
    kr->op = op;
    kr->k = k;
    kr->family = family;
    kr->k_per_split = (int)(depth / k.split);
    kr->kdepth = (int)depth;
    kr->smem = smem_bytes(k, family, op->out_f32, batched);
    kr->flops = 2.0 * (double)op->batch * (double)op->rows * (double)op->cols * (double)op->flop_depth;
    int st = OPEVO_OK;
    const int swz = swizzle_bytes(k.bk);
    const uint32_t atom_k = (uint32_t)(swz / 2);
    if (family == 1) {
        const int32_t* c = op->d.conv;
        int N = c[0], H = c[2], W = c[3], KH = c[5], KW = c[6], S = c[7], P = c[8];
        int HO = (H + 2 * P - KH) / S + 1, WO = (W + 2 * P - KW) / S + 1;
        const int hkw = halo_kw(k, family);
        const int CP = op->cpad;                          // Cin padded to 16 (kernel layout)
        // per-CTA tile: TILE_N images x TILE_H lines of LINE tile rows; a
        // CTA pair holds 2 x TILE_N images
        const int line_rows = hkw ? 16 : k.line ? k.line : k.tile_w;
        const int bm_cta = bm_cta_of(k);
        const int tile_n = bm_cta / (k.tile_h * line_rows);
        const int pair_n = tile_n * k.cg;
        if (hkw && (hkw != KW || k.split != 1 || P >= KW || S != 1)) {
            put_err(err, errlen, "halo lines of %d pixels need a %d-wide stride-1 filter (this one is %d wide, "
                    "stride %d)", k.tile_w, hkw, KW, S);
            delete kr;
            return OPEVO_INVALID_CONFIG;
        }
        if (tile_n < 1 || CP % k.bk || HO % k.tile_h || WO % k.tile_w || N % pair_n ||
            line_rows * S > 256 || k.tile_h * S > 256) {
            put_err(err, errlen, "conv tiling (n%d h%d w%d line %d, BK %d, stride %d) does not divide the problem",
                    pair_n, k.tile_h, k.tile_w, line_rows, k.bk, S);
            delete kr;
            return OPEVO_INVALID_CONFIG;
        }
        kr->geom = ConvGeomHost{CP, HO, WO, KW, P, CP / k.bk, S};
        uint64_t dims[4] = {(uint64_t)CP, (uint64_t)W, (uint64_t)H, (uint64_t)N};
        uint64_t strides[3] = {(uint64_t)CP * 2, (uint64_t)CP * W * 2, (uint64_t)CP * W * H * 2};
        // halo lines: 16 input pixels per line (TILE_W outputs + KW - 1 halo);
        // stride S: the box traverses S x the pixels with element stride S
        uint32_t box[4] = {atom_k, (uint32_t)(line_rows * S), (uint32_t)(k.tile_h * S), (uint32_t)tile_n};
        uint32_t es[4] = {1, (uint32_t)S, (uint32_t)S, 1};
        st = encode_map(&kr->tma_a, op->a, 4, dims, strides, box, swz, err, errlen, 0, es);
        if (b_resident(k, family)) {
            // resident weight panel: atom view {64, Cout, K/64}, one box {64, BN, K/64}
            const uint64_t d = (uint64_t)depth;
            const size_t panel = (size_t)k.bn * d * 2;
            if (!st && (op->cols != k.bn || d / 64 > 256 || kr->smem + 768 + panel > (size_t)ctx->smem_optin)) {
                put_err(err, errlen, "resident weights need BN = Cout (%lld) and a %zu B panel that fits",
                        (long long)op->cols, panel);
                st = OPEVO_INVALID_CONFIG;
            }
            uint64_t bd[3] = {64, (uint64_t)op->cols, d / 64};
            uint64_t bs[2] = {d * 2, 128};
            uint32_t bb[3] = {64, (uint32_t)k.bn, (uint32_t)(d / 64)};
            if (!st) st = encode_map(&kr->tma_b, op->b, 3, bd, bs, bb, 128, err, errlen);
            kr->smem += 768 + panel;    // 1 KB barrier block before the panel (BRES_OFF)
        } else if (hkw && !(getenv("OPEVO_WBOX") && getenv("OPEVO_WBOX")[0] == '0')) {
            // halo lines: one box per filter row holds its KW weight tiles,
            // every 64-channel atom of the K block -- view {64, Cout, Cin/64,
            // KH*KW} (W is [Cout][KH][KW][Cin]), box {64, BN/cg, BK/64, KW}
            uint64_t bd[4] = {64, (uint64_t)op->cols, (uint64_t)(CP / 64), (uint64_t)(KH * KW)};
            uint64_t bs[3] = {(uint64_t)depth * 2, 128, (uint64_t)CP * 2};
            uint32_t bb[4] = {64, (uint32_t)(k.bn / k.cg), (uint32_t)(k.bk / 64), (uint32_t)hkw};
            if (!st) st = encode_map(&kr->tma_b, op->b, 4, bd, bs, bb, 128, err, errlen);
        } else {
            uint64_t bd[2] = {(uint64_t)depth, (uint64_t)op->cols};
            uint64_t bs[1] = {(uint64_t)depth * 2};
            uint32_t bb[2] = {atom_k, (uint32_t)(k.bn / k.cg)};     // a CTA pair splits B's rows
            if (!st) st = encode_map(&kr->tma_b, op->b, 2, bd, bs, bb, swz, err, errlen);
        }
        if (!st) {
            // output NHWC {Cout, Wo, Ho, N}; a 32-pixel epilogue chunk of the
            // TILE_N x TILE_H x TILE_W tile is the box {EPI_COLS, bw, bh, bn}
            // (halo / padded lines: one box per line, {EPI_COLS, TILE_W, 1, 1};
            // the chunk's junk rows are never stored)
            const bool lines = hkw || k.line;
            const int ob = op->out_f32 ? 4 : 2, ec = epi_cols(k, family, op->out_f32, batched);
            const int bw = lines ? k.tile_w : std::min(k.tile_w, 32);
            const int bh = lines ? 1 : k.tile_w >= 32 ? 1 : std::min(k.tile_h, 32 / k.tile_w);
            const int bn = lines ? 1 : k.tile_w * k.tile_h >= 32 ? 1 : 32 / (k.tile_w * k.tile_h);
            if (!lines && (bw * bh * bn != 32 || k.tile_w % bw || k.tile_h % bh || tile_n % bn)) {
                put_err(err, errlen, "conv tile %dx%d cannot be stored in 32-pixel boxes", k.tile_h, k.tile_w);
                st = OPEVO_INVALID_CONFIG;
            } else {
                const int co = c[4];
                uint64_t cd[4] = {(uint64_t)co, (uint64_t)WO, (uint64_t)HO, (uint64_t)N};
                uint64_t cs[3] = {(uint64_t)co * ob, (uint64_t)co * WO * ob, (uint64_t)co * WO * HO * ob};
                uint32_t cb[4] = {(uint32_t)ec, (uint32_t)bw, (uint32_t)bh, (uint32_t)bn};
                st = encode_map(&kr->tma_c, op->c, 4, cd, cs, cb, ec * ob, err, errlen, op->out_f32);
            }
        }
        kr->sched = SchedHost{(N / pair_n) * (HO / k.tile_h) * (WO / k.tile_w), (int)col_tiles, 1,
                              k.split, 0, 1, 0};
        if (hkw) kr->kdepth = KH * CP;      // the K loop runs over filter rows x channel blocks
    } else {
        const uint32_t a_rows = (uint32_t)(bm_cta_of(k) / k.cluster);
        const uint32_t b_rows = (uint32_t)(k.bn / k.cg);
        const uint32_t bpu = (uint32_t)std::max(1, k.bpu);     // batches per work unit
        if (bpu > 1 && (!batched || op->batch % bpu)) {
            put_err(err, errlen, "bpu=%u needs a BatchMatMul whose batch (%lld) it divides", bpu,
                    (long long)op->batch);
            delete kr;
            return OPEVO_INVALID_CONFIG;
        }
        if (fused_k(k)) {
            // "atom" views {64, rows, K/64 (, batch)}: one box per operand per
            // stage (mirrors FUSED_K in gemm_sm100.cuh)
            const int rank = batched ? 4 : 3;
            const uint64_t d = (uint64_t)depth;
            uint64_t ad[4] = {64, (uint64_t)op->rows, d / 64, (uint64_t)op->batch};
            uint64_t as[3] = {d * 2, 128, d * op->rows * 2};
            uint32_t ab[4] = {64, a_rows, (uint32_t)(k.bk / 64), bpu};
            uint64_t bd[4] = {64, (uint64_t)op->cols, d / 64, (uint64_t)op->batch};
            uint64_t bs[3] = {d * 2, 128, d * op->cols * 2};
            uint32_t bb[4] = {64, b_rows, (uint32_t)(k.bk / 64), bpu};
            st = encode_map(&kr->tma_a, op->a, rank, ad, as, ab, 128, err, errlen);
            if (!st) st = encode_map(&kr->tma_b, op->b, rank, bd, bs, bb, 128, err, errlen);
        } else {
            const int rank = batched ? 3 : 2;
            uint64_t ad[3] = {(uint64_t)depth, (uint64_t)op->rows, (uint64_t)op->batch};
            uint64_t as[2] = {(uint64_t)depth * 2, (uint64_t)depth * op->rows * 2};
            uint32_t ab[3] = {atom_k, a_rows, bpu};
            uint64_t bd[3] = {(uint64_t)depth, (uint64_t)op->cols, (uint64_t)op->batch};
            uint64_t bs[2] = {(uint64_t)depth * 2, (uint64_t)depth * op->cols * 2};
            uint32_t bb[3] = {atom_k, b_rows, bpu};
            st = encode_map(&kr->tma_a, op->a, rank, ad, as, ab, swz, err, errlen);
            if (!st) st = encode_map(&kr->tma_b, op->b, rank, bd, bs, bb, swz, err, errlen);
        }
        const int rank = batched ? 3 : 2;
        if (!st) {
            const int ob = op->out_f32 ? 4 : 2, ec = epi_cols(k, family, op->out_f32, batched);
            uint64_t cd[3] = {(uint64_t)op->cols, (uint64_t)op->rows, (uint64_t)op->batch};
            uint64_t cs[2] = {(uint64_t)op->cols * ob, (uint64_t)op->cols * op->rows * ob};
            uint32_t cb[3] = {(uint32_t)ec, 32, 1};
            st = encode_map(&kr->tma_c, op->c, rank, cd, cs, cb, ec * ob, err, errlen, op->out_f32);
        }
        kr->sched = SchedHost{(int)row_tiles, (int)(col_tiles / k.cluster), (int)(op->batch / bpu), k.split,
                              0, 1, 0};
    }
    const bool dsm = dsmem_split(k, family, batched);
    const int tsplit = tma_split(k, family, batched);
    const int clsz = k.cluster * k.cg * (dsm ? k.split : 1);
    if (st) {
        delete kr;
        return st;
    }
    {
        double compile_ms_ = 0.0;
        int hit_ = 1;
        st = get_function(ctx, family, k, batched, op->out_f32, "opevo_gemm", kr->smem, &kr->fn, &compile_ms_,
                          &hit_, err, errlen);
        if (st) {
            delete kr;
            return st;
        }
        if (info) {
            info->compile_ms = compile_ms_;
            info->cache_hit = hit_;
        }
    }
    // grid: one cluster per unit, or (grid_mode 0) at most what is resident at
    // once, in which case CTAs loop over units (persistent schedule)
    {
        int per_sm = 1;
        if (g_cu.OccupancyMaxBlocks(&per_sm, kr->fn, 192, kr->smem) != CUDA_SUCCESS || per_sm < 1) per_sm = 1;
        // The occupancy API answers 1 CTA per SM for every tcgen05 kernel (it
        // does so for a 64-thread register-light one too), yet two
        // single-CTA instances whose shared memory fits twice do run side by
        // side (BMM1 128x64 BK 64, 2 stages: 262 -> 296 TFLOP/s with the
        // persistent grid at 296; profiles/round2/two_ctas_per_sm.txt).  For
        // single-CTA launches the residency is therefore counted from the
        // resources themselves: shared memory (+ static + the 1 KB per-CTA
        // reservation), registers (per-warp allocation in 256-register units),
        // threads, and below the TMEM columns.
        // (CTA pairs too: two pair clusters share an SM pair the same way)
        if ((clsz == 1 || (clsz == 2 && k.cg == 2 && k.cluster == 1)) && ctx->smem_per_sm > 0 &&
            ctx->regs_per_sm > 0) {
            int regs = 0, static_smem = 0;
            g_cu.FuncGetAttribute(&regs, CU_FUNC_ATTRIBUTE_NUM_REGS, kr->fn);
            g_cu.FuncGetAttribute(&static_smem, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, kr->fn);
            const long per_cta_smem = (long)kr->smem + static_smem + 1024;
            const int warps = 192 / 32;
            const long per_warp_regs = ((long)std::max(regs, 1) * 32 + 255) / 256 * 256;
            const int by_smem = (int)(ctx->smem_per_sm / per_cta_smem);
            const int by_regs = (int)(ctx->regs_per_sm / (per_warp_regs * warps));
            const int by_threads = 2048 / 192;
            per_sm = std::max(per_sm, std::min(std::min(by_smem, by_regs), std::min(by_threads, 32)));
        }
        static const int force_per_sm = getenv("OPEVO_FORCE_PER_SM") ? atoi(getenv("OPEVO_FORCE_PER_SM")) : 0;
        if (force_per_sm > 0) per_sm = force_per_sm;      // experiments only
        per_sm = std::min(per_sm, 512 / tmem_alloc_cols(k, family));
        const int capacity = std::max(1, (ctx->sm_count / clsz) * per_sm);
        SchedHost& sc = kr->sched;
        const int tiles = sc.row_tiles * sc.col_groups * sc.batches;
        sc.head_tiles = tiles;
        sc.tail_split = 1;
        // grid_mode 2: a persistent grid whose last wave would be partial cuts
        // the tiles of that wave into more K slices (stream-K style tail).
        // Measured slower than plain persistence on 4096^3 (the fp32 partials
        // cost more than the filled wave saves), so it is opt-in.
        if (k.grid_mode == 2 && k.split == 1 && tiles > capacity && tiles % capacity) {
            const int rem = tiles % capacity;
            int ts = 1;
            while (ts < 8 && 2 * ts * rem <= capacity && depth % ((int64_t)2 * ts * k.bk) == 0) ts *= 2;
            if (ts > 1) {
                sc.head_tiles = tiles - rem;
                sc.tail_split = ts;
            }
        }
        sc.units = sc.head_tiles * sc.split + (tiles - sc.head_tiles) * sc.split * sc.tail_split;
        // DSMEM split-K clusters each own exactly one unit (no persistence);
        // TMA split-K needs every slice resident at once (slice 0 waits for
        // the others): one wave or the configuration is infeasible
        if (tsplit && sc.units > capacity) {
            put_err(err, errlen, "TMA split-K needs one wave: %d units > %d resident CTAs", sc.units, capacity);
            delete kr;
            return OPEVO_INVALID_CONFIG;
        }
        const int clusters = (k.grid_mode == 1 || dsm || tsplit) ? sc.units / (dsm ? k.split : 1)
                                                                 : std::min(sc.units, capacity);
        kr->grid[0] = (unsigned)(clusters * clsz);
        kr->grid[1] = kr->grid[2] = 1;
        const int max_split = sc.split * sc.tail_split;
        if (max_split > 1 && !dsm) {
            const size_t slice = (size_t)op->batch * op->rows * op->cols * 4;
            st = ensure_ws(op, slice * max_split, (size_t)tiles * clsz * 4, err, errlen);
            if (!st && tsplit) st = encode_split_map(kr, tsplit, err, errlen);
            if (st) {
                delete kr;
                return st;
            }
        }
    }
    if (info) {
        info->load_ms = now_ms() - t0 - info->compile_ms;
        info->grid_ctas = (int32_t)(kr->grid[0] * kr->grid[1] * kr->grid[2]);
        info->smem_bytes = (int32_t)kr->smem;
    }
    *out = kr;
    return OPEVO_OK;
}

void opevo_kernel_release(opevo_kernel* k) { delete k; }

int opevo_kernel_run(opevo_kernel* k, char* err, size_t errlen) {
    if (!k) return OPEVO_ERR_ARG;
    opevo_ctx* ctx = k->op->ctx;
    g_cu.CtxSetCurrent(ctx->cu);
    int st = launch_kernel(k, err, errlen);
    if (st) return st;
    return sync_checked(ctx, "kernel", err, errlen);
}

}  // extern "C"

namespace {

// Enqueue the verification of one launch: poison C (NaN bytes, so a kernel
// that skips tiles fails), launch, compare against the reference into
// compare slot `slot` of ctx->cmp_buf (16 bytes each).  No synchronisation;
// see finish_check.
int enqueue_check(opevo_kernel* k, char* err, size_t errlen, int slot = 0, CUevent e0 = nullptr,
                  CUevent e1 = nullptr) {
    opevo_op* op = k->op;
    opevo_ctx* ctx = op->ctx;
    CU_TRY(ctx, g_cu.MemsetD8Async(op->c, 0xFF, op->c_bytes, ctx->stream), "poison C");
    if (e0) CU_TRY(ctx, g_cu.EventRecord(e0, ctx->stream), "event");
    int st = launch_kernel(k, err, errlen);
    if (st) return st;
    if (e1) CU_TRY(ctx, g_cu.EventRecord(e1, ctx->stream), "event");
    CUdeviceptr out = ctx->cmp_buf + 16 * (CUdeviceptr)slot;
    CU_TRY(ctx, g_cu.MemsetD8Async(out, 0, 16, ctx->stream), "zero compare");
    uint64_t n = (uint64_t)op->batch * op->rows * op->cols;
    int c_f32 = op->out_f32;
    void* args[] = {&op->c, &op->ref, &n, &c_f32, &out};
    // four outputs per thread-step, a few steps per thread, one atomic set per block
    const unsigned cgrid = (unsigned)std::min<uint64_t>((uint64_t)ctx->sm_count * 4,
                                                        std::max<uint64_t>(1, (n / 4 + 255) / 256));
    return launch_simple(ctx, ctx->k_compare, cgrid, 256, args, err, errlen);
}

// Judge one compare slot {max|C-R|, max|R|, non-finite count}.
int judge(const uint32_t* res, double tol, double* rel_err, char* err, size_t errlen) {
    float md, mr;
    memcpy(&md, &res[0], 4);
    memcpy(&mr, &res[1], 4);
    double rel = res[2] ? INFINITY : (mr > 0 ? (double)md / (double)mr : (double)md);
    if (rel_err) *rel_err = rel;
    if (!(rel <= tol)) {
        put_err(err, errlen, "output mismatch: rel err %.3g > tol %.3g (%u non-finite)", rel, tol, res[2]);
        return OPEVO_VERIFY_FAILED;
    }
    return OPEVO_OK;
}

// After the stream has drained: read the comparison and judge it.
int finish_check(opevo_kernel* k, double tol, double* rel_err, char* err, size_t errlen) {
    opevo_ctx* ctx = k->op->ctx;
    uint32_t res[4] = {0, 0, 0, 0};
    CU_TRY(ctx, g_cu.MemcpyDtoH(res, ctx->cmp_buf, 12), "compare readback");
    return judge(res, tol, rel_err, err, errlen);
}

// Device-time budget per measurement (ctx->budget_ms, opevo_ctx_set_timing;
// default OPEVO_TIME_BUDGET_MS or 0.3): a one-launch estimate caps the
// repetitions of slow candidates at budget/estimate (min 5), so a 30 us
// instance costs 10 launches rather than 20 and a 10 ms one 5; the fast
// instances that decide the search keep all `reps`.  Once the measured time
// is device-bound (the trial pipeline's host work is overlapped), this
// budget sets the trial rate.
// A candidate whose single timed launch exceeds the whole per-trial budget.
bool slow_candidate(const opevo_ctx* ctx, float est_ms) {
    return ctx->budget_ms > 0 && est_ms > ctx->budget_ms;
}

int capped_reps(const opevo_ctx* ctx, int reps, float est_ms) {
    const double budget = ctx->budget_ms;
    if (budget > 0 && est_ms > 0 && est_ms * reps > budget) {
        // quantised to {reps, 16, 8, 5} so an instance has few distinct timed graphs
        const int want = std::max(std::min(reps, 5), (int)(budget / est_ms));
        const int steps[] = {16, 8, 5};
        int q = std::min(reps, 5);
        for (int v : steps)
            if (v <= want && v < reps) { q = v; break; }
        reps = q;
    }
    return reps;
}

// Straggler control (ctx->loser_ratio > 0): a verified candidate whose
// single-launch estimate exceeds loser_ratio x the fastest estimate verified
// on this operator so far cannot reach the top of the archive; it is timed
// with loser_reps back-to-back launches and no extra warm-up instead of the
// full measurement.  Its fitness stays a measured back-to-back time, only
// with fewer samples; the competitive candidates keep every repetition.
bool loser(const opevo_op* op, float est_ms) {
    const opevo_ctx* ctx = op->ctx;
    return ctx->loser_ratio > 0 && op->best_est_ms > 0 && est_ms > ctx->loser_ratio * op->best_est_ms;
}

// `reps` back-to-back launches timed with CUDA events on the library stream.
// The stream first parks on a device-side gate (opevo_gate polling a mapped
// host flag); the host enqueues e0, the launches and e1, then opens the
// gate, so the launches run with no host gaps (PDL between them, as in a
// CUDA graph) without paying for graph instantiation on every trial.
// Segments of at most 64 launches keep the launch queue from filling while
// the gate is closed.
int time_gated(opevo_kernel* k, int reps, double* total_ms, char* err, size_t errlen) {
    opevo_ctx* ctx = k->op->ctx;
    CUevent e0, e1;
    CU_TRY(ctx, g_cu.EventCreate(&e0, CU_EVENT_DEFAULT), "event");
    CUresult r = g_cu.EventCreate(&e1, CU_EVENT_DEFAULT);
    if (r != CUDA_SUCCESS) {
        g_cu.EventDestroy(e0);
        return fail_cu(ctx, r, "event", err, errlen);
    }
    int st = OPEVO_OK;
    double total = 0.0;
    for (int done = 0; done < reps && !st;) {
        const int n = std::min(64, reps - done);
        uint32_t seq = ++ctx->gate_seq;
        uint64_t timeout_ns = 2000000000ull;
        void* ga[] = {&ctx->gate_dev, &seq, &timeout_ns};
        st = launch_simple(ctx, ctx->k_gate, 1, 32, ga, err, errlen);
        r = CUDA_SUCCESS;
        if (!st) r = g_cu.EventRecord(e0, ctx->stream);
        for (int i = 0; i < n && !st && r == CUDA_SUCCESS; ++i) st = launch_kernel(k, err, errlen);
        if (!st && r == CUDA_SUCCESS) r = g_cu.EventRecord(e1, ctx->stream);
        __atomic_store_n(const_cast<uint32_t*>(ctx->gate_host), seq, __ATOMIC_SEQ_CST);   // open
        if (!st && r == CUDA_SUCCESS) r = g_cu.EventSynchronize(e1);
        float ms = 0.f;
        if (!st && r == CUDA_SUCCESS) r = g_cu.EventElapsedTime(&ms, e0, e1);
        if (!st && r != CUDA_SUCCESS) {
            st = fail_cu(ctx, r, "timed launches", err, errlen);
            if (st != OPEVO_ERR_STICKY) st = OPEVO_LAUNCH_ERROR;
        }
        total += ms;
        done += n;
    }
    g_cu.EventDestroy(e0);
    g_cu.EventDestroy(e1);
    if (st) {
        // a failed launch leaves the stream parked: drain it
        g_cu.StreamSynchronize(ctx->stream);
        return st;
    }
    *total_ms = total;
    return OPEVO_OK;
}

// `reps` launches captured (on the side stream, so this host work overlaps
// device work already queued on ctx->stream) into one executable graph.
int build_graph(opevo_kernel* k, int reps, CUgraphExec* out, char* err, size_t errlen,
                CUstream cap = nullptr) {
    opevo_ctx* ctx = k->op->ctx;
    if (!cap) cap = ctx->cap_stream;
    CUgraph g = nullptr;
    CU_TRY(ctx, g_cu.StreamBeginCapture(cap, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL), "capture");
    int st = OPEVO_OK;
    for (int i = 0; i < reps && !st; ++i) st = launch_kernel(k, err, errlen, cap);
    CUresult r = g_cu.StreamEndCapture(cap, &g);
    if (!st && r == CUDA_SUCCESS) r = g_cu.GraphInstantiate(out, g, 0);
    if (g) g_cu.GraphDestroy(g);
    if (st) return st;
    if (r != CUDA_SUCCESS) return fail_cu(ctx, r, "graph", err, errlen);
    return OPEVO_OK;
}

// The graph's launches back to back (PDL edges between them, as captured),
// timed with CUDA events on the library stream; the graph is uploaded first
// so the timed launch carries no first-launch setup.
int time_graph(opevo_kernel* k, CUgraphExec ge, double* total_ms, char* err, size_t errlen) {
    opevo_ctx* ctx = k->op->ctx;
    CUevent e0, e1;
    CU_TRY(ctx, g_cu.EventCreate(&e0, CU_EVENT_DEFAULT), "event");
    CUresult r = g_cu.EventCreate(&e1, CU_EVENT_DEFAULT);
    if (r == CUDA_SUCCESS) r = g_cu.GraphUpload(ge, ctx->stream);
    if (r == CUDA_SUCCESS) r = g_cu.EventRecord(e0, ctx->stream);
    if (r == CUDA_SUCCESS) r = g_cu.GraphLaunch(ge, ctx->stream);
    if (r == CUDA_SUCCESS) r = g_cu.EventRecord(e1, ctx->stream);
    if (r == CUDA_SUCCESS) r = g_cu.EventSynchronize(e1);
    float ms = 0.f;
    if (r == CUDA_SUCCESS) r = g_cu.EventElapsedTime(&ms, e0, e1);
    g_cu.EventDestroy(e0);
    g_cu.EventDestroy(e1);
    if (r != CUDA_SUCCESS) {
        int st = fail_cu(ctx, r, "timed graph", err, errlen);
        return st == OPEVO_ERR_STICKY ? st : OPEVO_LAUNCH_ERROR;
    }
    *total_ms = ms;
    return OPEVO_OK;
}

// Cold-L2 timing: a 2x-L2 read pass (opevo_flush: clean lines only, so the
// timed launch pays no write-backs) before every launch, each timed alone.
int time_flushed(opevo_kernel* k, int reps, double* total_ms, char* err, size_t errlen) {
    opevo_ctx* ctx = k->op->ctx;
    if (!ctx->flush_buf) {
        ctx->flush_bytes = (size_t)256 << 20;   // 2x the 126 MB L2
        CU_TRY(ctx, g_cu.MemAlloc(&ctx->flush_buf, ctx->flush_bytes), "alloc flush buffer");
    }
    CUevent e0, e1;
    CU_TRY(ctx, g_cu.EventCreate(&e0, CU_EVENT_DEFAULT), "event");
    CU_TRY(ctx, g_cu.EventCreate(&e1, CU_EVENT_DEFAULT), "event");
    uint64_t n16 = ctx->flush_bytes / 16;
    double total = 0.0;
    int st = OPEVO_OK;
    for (int i = 0; i < reps; ++i) {
        unsigned salt = (unsigned)i;
        void* fa[] = {&ctx->flush_buf, &n16, &salt};
        st = launch_simple(ctx, ctx->k_flush, (unsigned)ctx->sm_count * 4, 512, fa, err, errlen);
        if (!st) st = g_cu.EventRecord(e0, ctx->stream) == CUDA_SUCCESS ? OPEVO_OK : OPEVO_ERR_CUDA;
        if (!st) st = launch_kernel(k, err, errlen);
        if (!st) st = g_cu.EventRecord(e1, ctx->stream) == CUDA_SUCCESS ? OPEVO_OK : OPEVO_ERR_CUDA;
        if (!st) st = sync_checked(ctx, "timed launch", err, errlen);
        float ms = 0.f;
        if (!st) g_cu.EventElapsedTime(&ms, e0, e1);
        if (st) break;
        total += ms;
    }
    g_cu.EventDestroy(e0);
    g_cu.EventDestroy(e1);
    if (st) return st;
    *total_ms = total;
    return OPEVO_OK;
}

// Warm-up launches plus a one-launch estimate between events; the caller
// synchronises (alone or together with an enqueued check).
int enqueue_warmup_estimate(opevo_kernel* k, int warmup, CUevent e0, CUevent e1, char* err,
                            size_t errlen) {
    opevo_ctx* ctx = k->op->ctx;
    for (int i = 0; i < warmup; ++i) {
        int st = launch_kernel(k, err, errlen);
        if (st) return st;
    }
    CU_TRY(ctx, g_cu.EventRecord(e0, ctx->stream), "event");
    int st = launch_kernel(k, err, errlen);
    if (st) return st;
    CU_TRY(ctx, g_cu.EventRecord(e1, ctx->stream), "event");
    return OPEVO_OK;
}

// Timing modes (the `flush_l2` argument of the ABI):
//   0  R back-to-back launches in one CUDA graph (L2 warm) -- the fitness
//   1  a 2x-L2 write before every launch, each launch timed (cold L2)
//   2  R back-to-back stream launches behind a device gate (no graph)
//
// One trial = phase A (the verified launch, timed by events, + the compare;
// one synchronisation) then, for candidates faster than the device budget,
// phase B: warm-up launches and the timed launches.  A candidate whose
// verified launch already exceeds the budget is measured by that launch
// alone: it is far from competitive, and on a large operator a bad tile can
// take milliseconds per launch -- with several GPUs evaluating one trial
// each per generation such a straggler would set the generation time.
// Without a check (tol < 0) an untimed-check estimate launch plays the same
// role.  In mode 0 the graph is captured and instantiated while phase A runs
// on the device.
int check_and_time(opevo_kernel* k, double tol, double* rel_err, int warmup, int reps, int mode,
                   double* ms_per_launch, char* err, size_t errlen, bool budgeted) {
    opevo_ctx* ctx = k->op->ctx;
    int st = OPEVO_OK;
    CUgraphExec ge = nullptr;
    int graph_reps = 0;
    CUevent e0, e1;
    CU_TRY(ctx, g_cu.EventCreate(&e0, CU_EVENT_DEFAULT), "event");
    CU_TRY(ctx, g_cu.EventCreate(&e1, CU_EVENT_DEFAULT), "event");
    float est = 0.f;
    if (tol >= 0) st = enqueue_check(k, err, errlen, 0, e0, e1);
    else          st = enqueue_warmup_estimate(k, 0, e0, e1, err, errlen);
    if (!st && mode == 0 && ms_per_launch) {
        st = build_graph(k, reps, &ge, err, errlen);
        graph_reps = reps;
    }
    if (!st) st = sync_checked(ctx, "check", err, errlen);
    if (!st) {
        CUresult r = g_cu.EventElapsedTime(&est, e0, e1);
        if (r != CUDA_SUCCESS) st = fail_cu(ctx, r, "estimate", err, errlen);
    }
    g_cu.EventDestroy(e0);
    g_cu.EventDestroy(e1);
    if (!st && tol >= 0) st = finish_check(k, tol, rel_err, err, errlen);
    if (st || !ms_per_launch) {
        if (ge) g_cu.GraphExecDestroy(ge);
        return st;
    }
    if (budgeted && slow_candidate(ctx, est)) {
        if (ge) g_cu.GraphExecDestroy(ge);
        *ms_per_launch = est;
        return OPEVO_OK;
    }
    if (budgeted) reps = capped_reps(ctx, reps, est);
    for (int i = 0; i + 1 < warmup && !st; ++i) st = launch_kernel(k, err, errlen);
    double total = 0.0;
    if (!st && mode == 0) {
        if (reps != graph_reps) {
            g_cu.GraphExecDestroy(ge);
            ge = nullptr;
            st = build_graph(k, reps, &ge, err, errlen);
        }
        if (!st) st = time_graph(k, ge, &total, err, errlen);
        if (!st) k->launches += reps;
    } else if (!st && mode == 1) {
        st = time_flushed(k, reps, &total, err, errlen);
    } else if (!st) {
        st = time_gated(k, reps, &total, err, errlen);
    }
    if (ge) g_cu.GraphExecDestroy(ge);
    if (st) return st;
    *ms_per_launch = total / reps;
    return OPEVO_OK;
}

}  // namespace

extern "C" {

int opevo_kernel_check(opevo_kernel* k, double tol, double* rel_err, char* err, size_t errlen) {
    if (!k) return OPEVO_ERR_ARG;
    opevo_ctx* ctx = k->op->ctx;
    g_cu.CtxSetCurrent(ctx->cu);
    int st = fresh_reference(k->op, err, errlen);
    if (!st) st = enqueue_check(k, err, errlen);
    if (!st) st = sync_checked(ctx, "check", err, errlen);
    if (!st) st = finish_check(k, tol < 0 ? 0.0 : tol, rel_err, err, errlen);
    return st;
}

int opevo_kernels_time_rotating(opevo_kernel* const* ks, int n, int warmup, int reps, double* ms_per_launch,
                                char* err, size_t errlen) {
    if (!ks || n < 1 || reps < 1 || warmup < 0 || !ms_per_launch) return OPEVO_ERR_ARG;
    for (int i = 0; i < n; ++i)
        if (!ks[i] || ks[i]->op->ctx != ks[0]->op->ctx) return OPEVO_ERR_ARG;
    opevo_ctx* ctx = ks[0]->op->ctx;
    g_cu.CtxSetCurrent(ctx->cu);
    CUgraph g = nullptr;
    CUgraphExec ge = nullptr;
    CU_TRY(ctx, g_cu.StreamBeginCapture(ctx->cap_stream, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL), "capture");
    int st = OPEVO_OK;
    for (int i = 0; i < reps && !st; ++i) st = launch_kernel(ks[i % n], err, errlen, ctx->cap_stream);
    CUresult r = g_cu.StreamEndCapture(ctx->cap_stream, &g);
    if (!st && r == CUDA_SUCCESS) r = g_cu.GraphInstantiate(&ge, g, 0);
    if (g) g_cu.GraphDestroy(g);
    if (st) return st;
    if (r != CUDA_SUCCESS) return fail_cu(ctx, r, "graph", err, errlen);
    double total = 0.0;
    // warm-up passes of the whole cycle (module, instruction caches, TLBs);
    // they do not warm the L2 for the timed pass: every copy is evicted again
    // before the cycle comes back to it
    for (int w = 0; w < warmup && !st; ++w) {
        r = g_cu.GraphLaunch(ge, ctx->stream);
        if (r != CUDA_SUCCESS) st = fail_cu(ctx, r, "graph", err, errlen);
    }
    if (!st) st = time_graph(ks[0], ge, &total, err, errlen);
    if (!st) st = sync_checked(ctx, "rotating timing", err, errlen);
    g_cu.GraphExecDestroy(ge);
    if (st) return st;
    for (int i = 0; i < reps; ++i) ks[i % n]->launches += warmup + 1;
    *ms_per_launch = total / reps;
    return OPEVO_OK;
}

int opevo_kernel_time(opevo_kernel* k, int warmup, int reps, int flush_l2, double* ms_per_launch, char* err,
                      size_t errlen) {
    if (!k || reps < 1 || !ms_per_launch) return OPEVO_ERR_ARG;
    g_cu.CtxSetCurrent(k->op->ctx->cu);
    // an explicit measurement: exactly `reps` launches (the per-trial device
    // budget applies to the trial paths only)
    return check_and_time(k, -1.0, nullptr, warmup, reps, flush_l2, ms_per_launch, err, errlen, false);
}

int opevo_trial(opevo_ctx* ctx, opevo_op* op, const int32_t* knobs, int nknobs, int warmup, int reps,
                int flush_l2, double tol, opevo_trial_result* res, char* err, size_t errlen) {
    if (!res || reps < 1) return OPEVO_ERR_ARG;
    memset(res, 0, sizeof *res);
    opevo_kernel* k = nullptr;
    int st = opevo_kernel_get(ctx, op, knobs, nknobs, &k, res, err, errlen);
    if (st) return st;
    double rel = 0.0, ms = 0.0;
    st = fresh_reference(op, err, errlen);
    if (!st) st = check_and_time(k, tol < 0 ? 0.0 : tol, &rel, warmup, reps, flush_l2, &ms, err, errlen, true);
    res->rel_err = rel;
    if (!st) {
        res->ms = ms;
        res->tflops = ms > 0 ? k->flops / (ms * 1e-3) / 1e12 : 0.0;
    }
    res->launches = k->launches;
    opevo_kernel_release(k);
    return st;
}

int opevo_trial_batch(opevo_ctx* ctx, opevo_op* op, const int32_t* knobs, int nknobs, int count,
                      int warmup, int reps, int flush_l2, double tol, opevo_trial_result* res,
                      int32_t* status, char* msgs, size_t msg_stride, char* err, size_t errlen) {
    if (!ctx || !op || !knobs || !res || !status || count < 0 || count > OPEVO_MAX_BATCH || reps < 1)
        return OPEVO_ERR_ARG;
    const int mode = flush_l2;
    g_cu.CtxSetCurrent(ctx->cu);
    if (int rst = fresh_reference(op, err, errlen)) return rst;
    static const bool prof = getenv("OPEVO_PROFILE_BATCH") != nullptr;
    double tp[8] = {now_ms(), 0, 0, 0, 0, 0, 0, 0};
    std::vector<opevo_kernel*> ks(count, nullptr);
    std::vector<CUgraphExec> ge(count, nullptr);
    std::vector<int> greps(count, 0);
    // every graph built here joins the operand's cache (bounded: past 2048
    // entries new graphs are destroyed instead; destroying executable graphs
    // costs device round trips, so the cache is never flushed wholesale)
    auto remember = [&](int i) {
        if (!ge[i] || !ks[i]) return;
        const std::string key = graph_key(ks[i]->k, greps[i]);
        auto it = op->graphs.find(key);
        if (it == op->graphs.end() && op->graphs.size() < 2048) {
            op->graphs.emplace(key, ge[i]);
        } else if (it == op->graphs.end() || it->second != ge[i]) {
            g_cu.GraphExecDestroy(ge[i]);
        }
        ge[i] = nullptr;
    };
    std::vector<CUevent> ev(4 * (size_t)count, nullptr);   // per trial: est0, est1, t0, t1
    auto msg = [&](int i) -> char* { return msgs ? msgs + (size_t)i * msg_stride : nullptr; };
    auto mlen = [&]() -> size_t { return msgs ? msg_stride : 0; };
    int fatal = OPEVO_OK;
    for (int i = 0; i < count; ++i) {
        memset(&res[i], 0, sizeof res[i]);
        if (msg(i) && mlen()) msg(i)[0] = 0;
        status[i] = opevo_kernel_get(ctx, op, knobs + (size_t)i * nknobs, nknobs, &ks[i], &res[i], msg(i), mlen());
        if (status[i] < 0) { fatal = status[i]; break; }
    }
    tp[1] = now_ms();
    // (host pool) capture + instantiate every bound instance's timed graph,
    // in parallel, while this thread runs phase A
    std::vector<int> gst(count, OPEVO_OK);
    std::vector<std::string> gmsg(count);
    bool pooled = false;
    // OPEVO_NO_POOL=1: build the graphs on this thread (profilers that do not
    // follow stream capture on other threads, e.g. an ncu launch list)
    static const bool no_pool = getenv("OPEVO_NO_POOL") != nullptr;
    if (!fatal && mode == 0 && !no_pool) {
        if (!ctx->pool) {
            const int nw = 6;
            for (int w = 0; w < nw; ++w) {
                CUstream st_ = nullptr;
                if (g_cu.StreamCreate(&st_, CU_STREAM_NON_BLOCKING) != CUDA_SUCCESS) break;
                ctx->pool_streams.push_back(st_);
            }
            if (!ctx->pool_streams.empty()) {
                ctx->pool.reset(new HostPool());
                ctx->pool->start((int)ctx->pool_streams.size(), ctx->cu);
            }
        }
        if (ctx->pool) {
            std::vector<std::function<void(int)>> tasks;
            for (int i = 0; i < count; ++i) {
                if (status[i] != OPEVO_OK) continue;
                greps[i] = reps;
                auto hit = op->graphs.find(graph_key(ks[i]->k, reps));
                if (hit != op->graphs.end()) {          // captured by an earlier trial
                    ge[i] = hit->second;
                    continue;
                }
                tasks.push_back([&, i](int w) {
                    char e[512] = {0};
                    gst[i] = build_graph(ks[i], reps, &ge[i], e, sizeof e, ctx->pool_streams[w]);
                    if (gst[i]) gmsg[i] = e;
                });
            }
            ctx->pool->submit(std::move(tasks));
            pooled = true;
        }
    }
    // phase A (device): for every bound instance, the poisoned check launch
    // + compare into its slot, warm-ups and a one-launch estimate -- unless
    // the instance was verified on these operands by an earlier trial
    // (`op->verified`); such a trial skips the check and is re-timed only
    std::vector<char> cached(count, 0);
    std::vector<std::string> vkey(count);
    std::vector<int> nreps(count, reps);
    // warm-up launches before the timed ones: the check launch counts as one,
    // a re-timed (cached) instance gets its `warmup` in full; losers (see
    // loser()) get only what their first timed launch needs
    std::vector<int> nwarm(count, 0);
    std::vector<float> est_of(count, 0.f);             // one-launch estimate per trial (ms)
    auto plan = [&](int i, float est) {
        est_of[i] = est;
        if (loser(op, est)) {
            nreps[i] = std::min(reps, ctx->loser_reps);
            nwarm[i] = cached[i] ? 1 : 0;
        } else {
            nreps[i] = capped_reps(ctx, reps, est);
            nwarm[i] = std::max(0, warmup - 1 + cached[i]);
        }
    };
    // Gated stream timing (mode 2): each trial's warm-ups and timed launches
    // (between its own events) are queued behind a device gate of at most 64
    // launches, so the launch queue never fills while a gate holds the
    // stream and no host gap falls inside a measurement.
    bool gate_open = false;
    int in_gate = 0, gated_trials = 0;
    uint32_t seq = 0;
    auto open_gate = [&]() -> int {
        seq = ++ctx->gate_seq;
        uint64_t timeout_ns = 2000000000ull;
        void* ga[] = {&ctx->gate_dev, &seq, &timeout_ns};
        int gst2 = launch_simple(ctx, ctx->k_gate, 1, 32, ga, err, errlen);
        gate_open = gst2 == OPEVO_OK;
        in_gate = 0;
        return gst2;
    };
    auto release = [&]() {
        if (gate_open) __atomic_store_n(const_cast<uint32_t*>(ctx->gate_host), seq, __ATOMIC_SEQ_CST);
        gate_open = false;
    };
    // The first gate of a batch opens once `lead` timed launches of its
    // trial are queued behind it (OPEVO_GATE_LEAD, default 6; 0 = after the
    // whole trial): queueing a launch takes the host ~2 us and running one
    // takes the device longer (>= 4 us here), so the host stays ahead of the
    // device from there on and no host gap falls inside the measurement,
    // while the device no longer idles through the whole trial's enqueue
    // (0.04 ms of a one-trial batch: the per-rank case on 8 GPUs).
    static const int lead = [] {
        const char* v = getenv("OPEVO_GATE_LEAD");
        return v ? std::max(0, atoi(v)) : 6;
    }();
    auto enqueue_timed = [&](int i) -> int {
        const int need = nwarm[i] + nreps[i];
        // the first gate holds one trial, so the device starts while the
        // host queues the rest (queueing a trial takes less host time than
        // running it); a trial never straddles two gates
        if (gate_open && (in_gate + need > 64 || gated_trials == 1)) release();
        const bool first_gate = !gate_open && gated_trials == 0;
        if (!gate_open) {
            const int gst2 = open_gate();
            if (gst2) return gst2 < 0 ? gst2 : OPEVO_ERR_CUDA;
        }
        // only for launches short enough that the host outpaces them
        const bool early = first_gate && lead > 0 && est_of[i] >= 0.004f;
        int st2 = OPEVO_OK;
        for (int w = 0; w < nwarm[i] && !st2; ++w) st2 = launch_kernel(ks[i], msg(i), mlen());
        if (!st2 && g_cu.EventRecord(ev[4 * i + 2], ctx->stream) != CUDA_SUCCESS) st2 = OPEVO_ERR_CUDA;
        for (int r = 0; r < nreps[i] && !st2; ++r) {
            st2 = launch_kernel(ks[i], msg(i), mlen());
            if (early && r + 1 == lead) release();
        }
        if (!st2 && g_cu.EventRecord(ev[4 * i + 3], ctx->stream) != CUDA_SUCCESS) st2 = OPEVO_ERR_CUDA;
        in_gate += need;
        ++gated_trials;
        return st2;
    };
    std::vector<char> early(count, 0);
    for (int i = 0; i < count && !fatal; ++i) {
        if (status[i] != OPEVO_OK) continue;
        int st = OPEVO_OK;
        for (int e = 0; e < 4 && !st; ++e)
            if (g_cu.EventCreate(&ev[4 * i + e], CU_EVENT_DEFAULT) != CUDA_SUCCESS) st = OPEVO_ERR_CUDA;
        vkey[i] = graph_key(ks[i]->k, 0);
        // OPEVO_NO_VERIFY_CACHE=1: check every trial (e.g. to project
        // per-rank costs, where each rank keeps its own record)
        static const bool no_vcache = getenv("OPEVO_NO_VERIFY_CACHE") != nullptr;
        cached[i] = (!no_vcache && op->verified.count(vkey[i])) ? 1 : 0;
        // the verified launch is bracketed by events: it is also the estimate
        if (!st && !cached[i]) st = enqueue_check(ks[i], msg(i), mlen(), i, ev[4 * i], ev[4 * i + 1]);
        if (!st && mode == 0 && !pooled) {
            greps[i] = reps;
            auto hit = op->graphs.find(graph_key(ks[i]->k, reps));
            if (hit != op->graphs.end()) ge[i] = hit->second;
            else st = build_graph(ks[i], reps, &ge[i], msg(i), mlen());
        }
        status[i] = st;
        if (st < 0) fatal = st;
    }
    // Instances verified by an earlier trial need no judging: in mode 2 their
    // timed launches are queued right behind the checks, so the device keeps
    // working through the check synchronisation and the judging below.
    if (!fatal && mode == 2) {
        for (int i = 0; i < count && !fatal; ++i) {
            if (status[i] != OPEVO_OK || !cached[i]) continue;
            const opevo_op::Verified& v = op->verified[vkey[i]];
            if (tol >= 0 && !(v.rel_err <= tol)) continue;       // judged (and failed) below
            plan(i, v.est_ms);
            status[i] = enqueue_timed(i);
            early[i] = 1;
            if (status[i] < 0) fatal = status[i];
        }
        release();
    }
    tp[2] = now_ms();
    if (pooled) {
        ctx->pool->wait();
        for (int i = 0; i < count; ++i) {
            if (status[i] != OPEVO_OK || gst[i] == OPEVO_OK) continue;
            status[i] = gst[i];
            if (msg(i) && mlen()) snprintf(msg(i), mlen(), "%s", gmsg[i].c_str());
            if (gst[i] < 0 && !fatal) fatal = gst[i];
        }
    }
    std::vector<uint32_t> cmp(4 * (size_t)std::max(count, 1), 0);
    tp[3] = now_ms();
    if (!fatal) {
        fatal = sync_checked(ctx, "batch check/warm-up", err, errlen);
        if (fatal == OPEVO_LAUNCH_ERROR) fatal = OPEVO_ERR_CUDA;
    }
    if (!fatal && count && g_cu.MemcpyDtoH(cmp.data(), ctx->cmp_buf, 16 * (size_t)count) != CUDA_SUCCESS)
        fatal = OPEVO_ERR_CUDA;
    // judge; candidates slower than the whole budget keep their verified
    // launch's time (no phase B); cap the repetitions of the rest
    std::vector<char> timed(count, 0);
    for (int i = 0; i < count && !fatal; ++i) {
        if (status[i] != OPEVO_OK) continue;
        float est = 0.f;
        if (cached[i]) {
            const opevo_op::Verified& v = op->verified[vkey[i]];
            res[i].rel_err = v.rel_err;
            res[i].verify_cached = 1;
            est = v.est_ms;
            if (tol >= 0 && !(v.rel_err <= tol)) {
                status[i] = OPEVO_VERIFY_FAILED;
                put_err(msg(i), mlen(), "rel err %.3e > tol %.1e (verified earlier)", v.rel_err, tol);
                continue;
            }
        } else {
            double rel = 0.0;
            status[i] = judge(&cmp[4 * (size_t)i], tol < 0 ? 0.0 : tol, &rel, msg(i), mlen());
            res[i].rel_err = rel;
            if (status[i] != OPEVO_OK) continue;
            g_cu.EventElapsedTime(&est, ev[4 * i], ev[4 * i + 1]);
            if (prof) fprintf(stderr, "[check %d] est %.4f ms\n", i, est);
            // slow candidates are timed by their verified launch itself, so
            // only fast ones are remembered (a repeat of a slow one re-checks)
            if (!slow_candidate(ctx, est) && tol >= 0) op->verified[vkey[i]] = opevo_op::Verified{rel, est};
        }
        if (slow_candidate(ctx, est)) {
            res[i].ms = est;
            timed[i] = 1;
            continue;
        }
        if (op->best_est_ms <= 0.f || est < op->best_est_ms) op->best_est_ms = est;
        if (!early[i]) plan(i, est);
        if (mode == 0 && nreps[i] != greps[i]) {
            remember(i);                                 // keep the full-length graph too
            greps[i] = nreps[i];
            auto hit = op->graphs.find(graph_key(ks[i]->k, nreps[i]));
            if (hit != op->graphs.end()) {
                ge[i] = hit->second;
            } else {
                status[i] = build_graph(ks[i], nreps[i], &ge[i], msg(i), mlen());
                if (status[i] < 0) fatal = status[i];
            }
        }
    }
    tp[4] = tp[5] = now_ms();
    // phase B: the timed launches of every verified instance, back to back,
    // each bracketed by its own events; one synchronisation at the end
    if (!fatal && mode == 0) {
        int last = -1;
        for (int i = 0; i < count; ++i) {
            if (status[i] != OPEVO_OK || timed[i]) continue;
            int wst = OPEVO_OK;
            for (int w = 0; w < nwarm[i] && !wst; ++w) wst = launch_kernel(ks[i], msg(i), mlen());
            if (wst) {
                status[i] = wst;
                if (wst < 0) { fatal = wst; break; }
                continue;
            }
            CUresult r = g_cu.GraphUpload(ge[i], ctx->stream);
            if (r == CUDA_SUCCESS) r = g_cu.EventRecord(ev[4 * i + 2], ctx->stream);
            if (r == CUDA_SUCCESS) r = g_cu.GraphLaunch(ge[i], ctx->stream);
            if (r == CUDA_SUCCESS) ks[i]->launches += nreps[i];
            if (r == CUDA_SUCCESS) r = g_cu.EventRecord(ev[4 * i + 3], ctx->stream);
            if (r != CUDA_SUCCESS) {
                status[i] = fail_cu(ctx, r, "timed graph", msg(i), mlen());
                if (status[i] < 0) { fatal = status[i]; break; }
                continue;
            }
            last = i;
        }
        tp[5] = now_ms();
        if (!fatal && last >= 0) {
            fatal = sync_checked(ctx, "batch timing", err, errlen);
            if (fatal == OPEVO_LAUNCH_ERROR) fatal = OPEVO_ERR_CUDA;
        }
        for (int i = 0; i < count && !fatal; ++i) {
            if (status[i] != OPEVO_OK || timed[i]) continue;
            float ms = 0.f;
            g_cu.EventElapsedTime(&ms, ev[4 * i + 2], ev[4 * i + 3]);
            res[i].ms = ms / nreps[i];
        }
    } else if (!fatal && mode == 2) {
        // every other verified instance's warm-ups and timed launches behind
        // the gates (the early ones are already queued); one synchronisation
        int last = -1;
        for (int i = 0; i < count && !fatal; ++i) {
            if (status[i] != OPEVO_OK || timed[i] || early[i]) continue;
            const int st2 = enqueue_timed(i);
            status[i] = st2;
            if (st2 < 0) fatal = st2;
            else if (!st2) last = i;
        }
        for (int i = 0; i < count; ++i)
            if (early[i] && status[i] == OPEVO_OK) last = i;
        tp[5] = now_ms();
        release();
        if (last >= 0 || fatal) {
            const int sst = sync_checked(ctx, "batch timing", err, errlen);
            if (!fatal && sst) fatal = sst == OPEVO_LAUNCH_ERROR ? OPEVO_ERR_CUDA : sst;
        }
        for (int i = 0; i < count && !fatal; ++i) {
            if (status[i] != OPEVO_OK || timed[i]) continue;
            float ms = 0.f;
            g_cu.EventElapsedTime(&ms, ev[4 * i + 2], ev[4 * i + 3]);
            res[i].ms = ms / nreps[i];
        }
    } else if (!fatal) {
        for (int i = 0; i < count && !fatal; ++i) {
            if (status[i] != OPEVO_OK || timed[i]) continue;
            for (int w = 0; w < nwarm[i] && status[i] == OPEVO_OK; ++w)
                status[i] = launch_kernel(ks[i], msg(i), mlen());
            if (status[i] != OPEVO_OK) {
                if (status[i] < 0) fatal = status[i];
                continue;
            }
            double total = 0.0;
            status[i] = mode == 1 ? time_flushed(ks[i], nreps[i], &total, msg(i), mlen())
                                  : time_gated(ks[i], nreps[i], &total, msg(i), mlen());
            if (status[i] < 0) fatal = status[i];
            else if (status[i] == OPEVO_OK) res[i].ms = total / nreps[i];
        }
    }
    for (int i = 0; i < count; ++i) {
        if (fatal && status[i] == OPEVO_OK) status[i] = fatal;
        if (status[i] == OPEVO_OK && res[i].ms > 0) res[i].tflops = ks[i]->flops / (res[i].ms * 1e-3) / 1e12;
        if (fatal) {                                     // nothing from a failed batch is kept
            if (ge[i] && !op->graphs.count(graph_key(ks[i]->k, greps[i]))) g_cu.GraphExecDestroy(ge[i]);
            ge[i] = nullptr;
        } else {
            remember(i);                                 // needs ks[i]: before the release
        }
        if (ks[i]) {
            res[i].launches = ks[i]->launches;
            opevo_kernel_release(ks[i]);
            ks[i] = nullptr;
        }
        for (int e = 0; e < 4; ++e)
            if (ev[4 * i + e]) g_cu.EventDestroy(ev[4 * i + e]);
    }
    if (fatal && err && errlen && !err[0]) put_err(err, errlen, "batch aborted (status %d)", fatal);
    if (prof) {
        tp[6] = now_ms();
        fprintf(stderr, "[batch %d] bind %.3f enqA %.3f poolwait %.3f syncA+judge %.3f enqB %.3f syncB+rest %.3f ms\n",
                count, tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4], tp[6] - tp[5]);
    }
    return fatal;
}

int opevo_op_preload(opevo_ctx* ctx, opevo_op* op, const int32_t* knobs, int nknobs, double* compile_ms,
                     int* cache_hit, char* err, size_t errlen) {
    if (!ctx || !op || !knobs) return OPEVO_ERR_ARG;
    if (ctx->poisoned) {
        put_err(err, errlen, "context poisoned by an earlier fault");
        return OPEVO_ERR_STICKY;
    }
    g_cu.CtxSetCurrent(ctx->cu);
    const int family = family_of(op->d);
    Knobs k = lib_knobs(family, knobs, nknobs);
    const int batched = op->d.kind == OPEVO_BATCHMATMUL ? 1 : 0;
    if (!knobs_compilable(family, k, err, errlen)) return OPEVO_INVALID_CONFIG;
    CUfunction fn = nullptr;
    double cms = 0.0;
    int hit = 1;
    int st = get_function(ctx, family, k, batched, family == 2 ? 1 : op->out_f32,
                          family == 2 ? "opevo_sgemm" : "opevo_gemm", 0, &fn, &cms, &hit, err, errlen);
    if (compile_ms) *compile_ms = cms;
    if (cache_hit) *cache_hit = hit;
    return st;
}

int opevo_ctx_set_timing(opevo_ctx* ctx, double budget_ms, double loser_ratio, int loser_reps) {
    if (!ctx || loser_reps < 1) return OPEVO_ERR_ARG;
    ctx->budget_ms = budget_ms;
    ctx->loser_ratio = loser_ratio;
    ctx->loser_reps = loser_reps;
    return OPEVO_OK;
}

static int flush_l2_enqueue(opevo_ctx* ctx, char* err, size_t errlen);

int opevo_ctx_flush_l2(opevo_ctx* ctx, char* err, size_t errlen) {
    if (!ctx) return OPEVO_ERR_ARG;
    const int st = flush_l2_enqueue(ctx, err, errlen);
    if (st) return st;
    return sync_checked(ctx, "flush", err, errlen);
}

int opevo_ctx_flush_l2_async(opevo_ctx* ctx, char* err, size_t errlen) {
    if (!ctx) return OPEVO_ERR_ARG;
    return flush_l2_enqueue(ctx, err, errlen);
}

static int flush_l2_enqueue(opevo_ctx* ctx, char* err, size_t errlen) {
    g_cu.CtxSetCurrent(ctx->cu);
    if (!ctx->flush_buf) {
        ctx->flush_bytes = (size_t)256 << 20;
        CU_TRY(ctx, g_cu.MemAlloc(&ctx->flush_buf, ctx->flush_bytes), "alloc flush buffer");
    }
    uint64_t n16 = ctx->flush_bytes / 16;
    unsigned salt = 0x5eed;
    void* fa[] = {&ctx->flush_buf, &n16, &salt};
    return launch_simple(ctx, ctx->k_flush, (unsigned)ctx->sm_count * 4, 512, fa, err, errlen);
}

int opevo_kernel_trace(opevo_kernel* k, uint64_t* host, size_t count, char* err, size_t errlen) {
    if (!k || !host) return OPEVO_ERR_ARG;
    opevo_op* op = k->op;
    opevo_ctx* ctx = op->ctx;
    g_cu.CtxSetCurrent(ctx->cu);
    const size_t ctas = (size_t)k->grid[0] * k->grid[1] * k->grid[2];
    const size_t per = ctas * 16;       // 16 stamps per CTA per launch
    // room for several launches in `host`: that many back-to-back launches
    // (PDL as in timing), each stamping its own block -> steady-state timeline
    const int nl = (int)std::max<size_t>(1, std::min<size_t>(8, count / per));
    const size_t bytes = per * nl * sizeof(uint64_t);
    CUdeviceptr buf = 0;
    CU_TRY(ctx, g_cu.MemAlloc(&buf, bytes), "alloc trace");
    CU_TRY(ctx, g_cu.MemsetD8(buf, 0, bytes), "zero trace");
    CUdeviceptr saved = op->ws;
    int st = OPEVO_OK;
    for (int i = 0; i < nl && !st; ++i) {
        op->ws = buf + (CUdeviceptr)(i * per * sizeof(uint64_t));   // stamps go through `ws`
        st = launch_kernel(k, err, errlen);
    }
    if (!st) st = sync_checked(ctx, "traced kernel", err, errlen);
    op->ws = saved;
    if (!st) {
        CUresult r = g_cu.MemcpyDtoH(host, buf, std::min(bytes, count * sizeof(uint64_t)));
        if (r != CUDA_SUCCESS) st = fail_cu(ctx, r, "read trace", err, errlen);
    }
    g_cu.MemFree(buf);
    return st;
}

void* opevo_host_alloc(size_t bytes) {
    load_driver();
    if (!g_cu.ok) return nullptr;
    void* p = nullptr;
    if (g_cu.MemAllocHost(&p, bytes) != CUDA_SUCCESS) return nullptr;
    return p;
}

void opevo_host_free(void* p) {
    if (p && g_cu.ok) g_cu.MemFreeHost(p);
}

}  // extern "C"
