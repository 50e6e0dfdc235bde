"""ctypes binding of ``libopevo.so`` (declared in ``include/opevo.h``).

This is the Python side of the drop-in boundary: the reference's objective
seam (``pkg/src/topotune/engine.py:264-310``) calls into the C ABI through
these wrappers.  There is no fallback -- if the library or the device is
missing, the calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libopevo.so")
DEFAULT_CACHE = os.path.join(HERE, "kernel_cache")

ABI_VERSION = 8

# status codes (opevo.h)
OK = 0
INVALID_CONFIG = 1
COMPILE_ERROR = 2
LAUNCH_ERROR = 3
VERIFY_FAILED = 4
ERR_NO_DEVICE = -1
ERR_NO_NVRTC = -2
ERR_STICKY = -3
ERR_ARG = -4
ERR_CUDA = -5

STATUS_NAMES = {OK: "ok", INVALID_CONFIG: "invalid_config", COMPILE_ERROR: "compile_error",
                LAUNCH_ERROR: "launch_error", VERIFY_FAILED: "verify_failed",
                ERR_NO_DEVICE: "no_device", ERR_NO_NVRTC: "no_nvrtc", ERR_STICKY: "sticky",
                ERR_ARG: "bad_argument", ERR_CUDA: "cuda_error"}

MATMUL, BATCHMATMUL, CONV2D = 0, 1, 2
BF16, F32, F32_TF32X3 = 0, 1, 2
FP32_OUT = (F32, F32_TF32X3)
NUM_KNOBS = 14
KNOB_NAMES = ("bm", "bn", "bk", "stages", "split", "cluster", "tile_h", "tile_w", "acc",
              "cta_group", "grid")

EXPORTS = (
    "opevo_abi_version", "opevo_compile", "opevo_kernel_key", "opevo_ctx_create",
    "opevo_ctx_destroy", "opevo_ctx_info", "opevo_op_prepare", "opevo_op_destroy",
    "opevo_op_sizes", "opevo_op_upload", "opevo_op_download", "opevo_op_read_inputs",
    "opevo_op_reference",
    "opevo_op_refresh_reference", "opevo_kernel_get", "opevo_kernel_release",
    "opevo_kernel_run", "opevo_kernel_check", "opevo_kernel_time", "opevo_kernels_time_rotating",
    "opevo_trial",
    "opevo_kernel_trace", "opevo_ctx_flush_l2", "opevo_ctx_flush_l2_async", "opevo_host_alloc", "opevo_host_free",
    "opevo_op_preload", "opevo_trial_batch", "opevo_ctx_set_timing",
    # native OpEvo proposal core (bound in native.py)
    "opevo_search_create", "opevo_search_destroy", "opevo_search_slots", "opevo_search_set_rng",
    "opevo_search_get_rng", "opevo_search_propose", "opevo_search_add_pending", "opevo_search_tell",
    "opevo_search_uniform_int", "opevo_search_random", "opevo_search_np_sum",
)
MAX_BATCH = 64


class OpDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dtype", C.c_int32), ("batch", C.c_int64),
                ("rows", C.c_int64), ("cols", C.c_int64), ("depth", C.c_int64),
                ("conv", C.c_int32 * 9), ("seed", C.c_uint64)]


class TrialResult(C.Structure):
    _fields_ = [("tflops", C.c_double), ("ms", C.c_double), ("rel_err", C.c_double),
                ("compile_ms", C.c_double), ("load_ms", C.c_double), ("cache_hit", C.c_int32),
                ("grid_ctas", C.c_int32), ("smem_bytes", C.c_int32), ("launches", C.c_int32),
                ("verify_cached", C.c_int32)]


class OpevoError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message

    @property
    def fatal(self) -> bool:
        return self.status < 0


_lib = None


def library_path() -> str:
    return os.environ.get("OPEVO_LIB", LIB_PATH)


def load() -> C.CDLL:
    """Load libopevo.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not os.path.exists(path):
        raise OSError(f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    P, I, D = C.c_void_p, C.c_int, C.c_double
    i32p, dp, cp, sz = C.POINTER(C.c_int32), C.POINTER(C.c_double), C.c_char_p, C.c_size_t
    sig = {
        "opevo_abi_version": (I, []),
        "opevo_compile": (I, [I, i32p, I, I, I, cp, dp, cp, sz]),
        "opevo_kernel_key": (I, [I, i32p, I, I, I, cp, sz]),
        "opevo_ctx_create": (I, [I, cp, C.POINTER(P), cp, sz]),
        "opevo_ctx_destroy": (None, [P]),
        "opevo_ctx_info": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
        "opevo_op_prepare": (I, [P, C.POINTER(OpDesc), C.POINTER(P), cp, sz]),
        "opevo_op_destroy": (None, [P]),
        "opevo_op_sizes": (I, [P, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz)]),
        "opevo_op_upload": (I, [P, P, P, cp, sz]),
        "opevo_op_download": (I, [P, P, sz, cp, sz]),
        "opevo_op_read_inputs": (I, [P, P, P, cp, sz]),
        "opevo_op_reference": (I, [P, C.POINTER(C.c_float), sz, cp, sz]),
        "opevo_op_refresh_reference": (I, [P, cp, sz]),
        "opevo_kernel_get": (I, [P, P, i32p, I, C.POINTER(P), C.POINTER(TrialResult), cp, sz]),
        "opevo_kernel_release": (None, [P]),
        "opevo_kernel_run": (I, [P, cp, sz]),
        "opevo_kernel_check": (I, [P, D, dp, cp, sz]),
        "opevo_kernel_time": (I, [P, I, I, I, dp, cp, sz]),
        "opevo_kernels_time_rotating": (I, [C.POINTER(P), I, I, I, dp, cp, sz]),
        "opevo_trial": (I, [P, P, i32p, I, I, I, I, D, C.POINTER(TrialResult), cp, sz]),
        "opevo_kernel_trace": (I, [P, C.POINTER(C.c_uint64), sz, cp, sz]),
        "opevo_ctx_flush_l2": (I, [P, cp, sz]),
        "opevo_ctx_flush_l2_async": (I, [P, cp, sz]),
        "opevo_ctx_set_timing": (I, [P, D, D, I]),
        "opevo_host_alloc": (P, [sz]),
        "opevo_host_free": (None, [P]),
        "opevo_op_preload": (I, [P, P, i32p, I, dp, C.POINTER(I), cp, sz]),
        "opevo_trial_batch": (I, [P, P, i32p, I, I, I, I, I, D, C.POINTER(TrialResult),
                                  C.POINTER(C.c_int32), cp, sz, cp, sz]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.opevo_abi_version() != ABI_VERSION:
        raise OSError("libopevo ABI version mismatch; rebuild")
    _lib = lib
    return lib


_KNOB_DEFAULTS = (128, 128, 64, 4, 1, 1, 1, 1, 1, 1, 0, 0, 1, 0)


def _knob_array(knobs) -> "C.Array":
    vals = list(knobs) + list(_KNOB_DEFAULTS[len(knobs):])
    return (C.c_int32 * NUM_KNOBS)(*vals[:NUM_KNOBS])


def _errbuf():
    return C.create_string_buffer(4096)


def _check(status: int, err) -> None:
    if status != OK:
        raise OpevoError(status, err.value.decode(errors="replace"))


def compile_kernel(family: int, knobs, batched: bool, out_f32: bool,
                   cache_dir: str = DEFAULT_CACHE) -> float:
    """NVRTC-compile one instance into the disk cache (no device needed).
    Returns compile ms (0.0 on a cache hit).  Thread-safe, releases the GIL."""
    lib = load()
    ms = C.c_double(0.0)
    err = _errbuf()
    st = lib.opevo_compile(family, _knob_array(knobs), NUM_KNOBS, int(batched), int(out_f32),
                           cache_dir.encode(), C.byref(ms), err, len(err))
    _check(st, err)
    return ms.value


def kernel_key(family: int, knobs, batched: bool, out_f32: bool) -> str:
    lib = load()
    buf = C.create_string_buffer(256)
    _check(lib.opevo_kernel_key(family, _knob_array(knobs), NUM_KNOBS, int(batched),
                                int(out_f32), buf, len(buf)), buf)
    return buf.value.decode()


@dataclass
class Trial:
    status: int
    tflops: float
    ms: float
    rel_err: float
    compile_ms: float
    load_ms: float
    cache_hit: int
    grid_ctas: int
    smem_bytes: int
    message: str
    launches: int = 0
    verify_cached: int = 0

    @property
    def ok(self) -> bool:
        return self.status == OK


class Device:
    """One CUDA context on one B200 (``opevo_ctx``)."""

    def __init__(self, device: int = 0, cache_dir: str = DEFAULT_CACHE):
        self.lib = load()
        self.device = device
        self.cache_dir = cache_dir
        os.makedirs(cache_dir, exist_ok=True)
        h = C.c_void_p()
        err = _errbuf()
        _check(self.lib.opevo_ctx_create(device, cache_dir.encode(), C.byref(h), err, len(err)), err)
        self.handle = h
        sm, smem, ma, mi = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        self.lib.opevo_ctx_info(h, C.byref(sm), C.byref(smem), C.byref(ma), C.byref(mi))
        self.sm_count, self.smem_optin, self.cc = sm.value, smem.value, (ma.value, mi.value)

    def close(self) -> None:
        if self.handle:
            self.lib.opevo_ctx_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_timing(self, budget_ms: float = 0.3, loser_ratio: float = 0.0, loser_reps: int = 5) -> None:
        """Trial timing policy (``opevo_ctx_set_timing``): per-trial device
        budget, and the straggler rule -- candidates slower than
        ``loser_ratio`` x the fastest verified one get ``loser_reps`` launches."""
        st = self.lib.opevo_ctx_set_timing(self.handle, budget_ms, loser_ratio, loser_reps)
        if st != OK:
            raise OpevoError(st, "bad timing policy")

    def flush_l2(self, wait: bool = True) -> None:
        """Evict L2 (read 2x its size); wait for it, or (wait=False) only
        enqueue it ahead of this context's later work."""
        err = _errbuf()
        fn = self.lib.opevo_ctx_flush_l2 if wait else self.lib.opevo_ctx_flush_l2_async
        _check(fn(self.handle, err, len(err)), err)

    def prepare(self, kind: int, dtype: int = BF16, batch: int = 1, rows: int = 0, cols: int = 0,
                depth: int = 0, conv=None, seed: int = 1234) -> "Operand":
        d = OpDesc()
        d.kind, d.dtype, d.batch, d.rows, d.cols, d.depth = kind, dtype, batch, rows, cols, depth
        for i, v in enumerate(conv or [0] * 9):
            d.conv[i] = int(v)
        d.seed = seed
        h = C.c_void_p()
        err = _errbuf()
        _check(self.lib.opevo_op_prepare(self.handle, C.byref(d), C.byref(h), err, len(err)), err)
        return Operand(self, h, d)

    def trial(self, op: "Operand", knobs, warmup: int = 3, reps: int = 20, flush_l2: bool = False,
              tol: float = 1e-2) -> Trial:
        res = TrialResult()
        err = _errbuf()
        st = self.lib.opevo_trial(self.handle, op.handle, _knob_array(knobs), NUM_KNOBS, warmup,
                                  reps, int(flush_l2), tol, C.byref(res), err, len(err))
        return Trial(st, res.tflops, res.ms, res.rel_err, res.compile_ms, res.load_ms,
                     res.cache_hit, res.grid_ctas, res.smem_bytes,
                     err.value.decode(errors="replace") if st != OK else "", res.launches)

    def trial_batch(self, op: "Operand", knob_list, warmup: int = 3, reps: int = 20,
                    flush_l2: int = 0, tol: float = 1e-2) -> list[Trial]:
        """Several trials with two host synchronisations in total (checks and
        warm-ups of all, then all timed launches).  A fatal (< 0) error raises
        OpevoError with the per-trial results attached as ``.trials``."""
        out: list[Trial] = []
        for lo in range(0, len(knob_list), MAX_BATCH):
            chunk = knob_list[lo:lo + MAX_BATCH]
            n = len(chunk)
            knobs = (C.c_int32 * (n * NUM_KNOBS))()
            for i, kn in enumerate(chunk):
                knobs[i * NUM_KNOBS:(i + 1) * NUM_KNOBS] = list(_knob_array(kn))
            res = (TrialResult * n)()
            status = (C.c_int32 * n)()
            stride = 512
            msgs = C.create_string_buffer(n * stride)
            err = _errbuf()
            st = self.lib.opevo_trial_batch(self.handle, op.handle, knobs, NUM_KNOBS, n, warmup, reps,
                                            int(flush_l2), tol, res, status, msgs, stride, err, len(err))
            trials = []
            for i in range(n):
                r = res[i]
                m = msgs.raw[i * stride:(i + 1) * stride].split(b"\0", 1)[0].decode(errors="replace")
                trials.append(Trial(status[i], r.tflops, r.ms, r.rel_err, r.compile_ms, r.load_ms,
                                    r.cache_hit, r.grid_ctas, r.smem_bytes,
                                    m if status[i] != OK else "", r.launches, r.verify_cached))
            out.extend(trials)
            if st != OK:
                e = OpevoError(st, err.value.decode(errors="replace"))
                e.trials = out
                raise e
        return out

    def preload(self, op: "Operand", knobs) -> tuple[int, float, int, str]:
        """Compile-or-read and load one instance's module (thread-safe; no
        launch).  Returns (status, compile_ms, cache_hit, message)."""
        cms, hit = C.c_double(), C.c_int()
        err = _errbuf()
        st = self.lib.opevo_op_preload(self.handle, op.handle, _knob_array(knobs), NUM_KNOBS,
                                       C.byref(cms), C.byref(hit), err, len(err))
        return st, cms.value, hit.value, err.value.decode(errors="replace") if st != OK else ""

    def kernel(self, op: "Operand", knobs) -> "Kernel":
        h = C.c_void_p()
        info = TrialResult()
        err = _errbuf()
        _check(self.lib.opevo_kernel_get(self.handle, op.handle, _knob_array(knobs), NUM_KNOBS,
                                         C.byref(h), C.byref(info), err, len(err)), err)
        return Kernel(self, h, info)


class Operand:
    """Prepared operator instance (``opevo_op``): operands + fp32 reference."""

    def __init__(self, dev: Device, handle, desc: OpDesc):
        self.dev, self.handle, self.desc = dev, handle, desc
        a, b, c = C.c_size_t(), C.c_size_t(), C.c_size_t()
        dev.lib.opevo_op_sizes(handle, C.byref(a), C.byref(b), C.byref(c))
        self.a_bytes, self.b_bytes, self.c_bytes = a.value, b.value, c.value

    def close(self) -> None:
        if self.handle:
            self.dev.lib.opevo_op_destroy(self.handle)
            self.handle = None

    def upload(self, a_ptr: int | None, b_ptr: int | None) -> None:
        err = _errbuf()
        _check(self.dev.lib.opevo_op_upload(self.handle, a_ptr, b_ptr, err, len(err)), err)

    def download(self, c_ptr: int, nbytes: int) -> None:
        err = _errbuf()
        _check(self.dev.lib.opevo_op_download(self.handle, c_ptr, nbytes, err, len(err)), err)

    def read_inputs(self, a_ptr: int | None, b_ptr: int | None) -> None:
        err = _errbuf()
        _check(self.dev.lib.opevo_op_read_inputs(self.handle, a_ptr, b_ptr, err, len(err)), err)

    def refresh_reference(self) -> None:
        err = _errbuf()
        _check(self.dev.lib.opevo_op_refresh_reference(self.handle, err, len(err)), err)

    def reference(self):
        import numpy as np

        n = self.c_bytes // (4 if self.desc.dtype in FP32_OUT else 2)
        out = np.empty(n, dtype=np.float32)
        err = _errbuf()
        _check(self.dev.lib.opevo_op_reference(
            self.handle, out.ctypes.data_as(C.POINTER(C.c_float)), n, err, len(err)), err)
        return out

    def output(self):
        """Kernel output as float32 numpy (bf16 widened)."""
        import numpy as np

        if self.desc.dtype in FP32_OUT:
            out = np.empty(self.c_bytes // 4, dtype=np.float32)
            self.download(out.ctypes.data, self.c_bytes)
            return out
        raw = np.empty(self.c_bytes // 2, dtype=np.uint16)
        self.download(raw.ctypes.data, self.c_bytes)
        return (raw.astype(np.uint32) << 16).view(np.float32)


class Kernel:
    """A bound launch plan (``opevo_kernel``)."""

    def __init__(self, dev: Device, handle, info: TrialResult):
        self.dev, self.handle, self.info = dev, handle, info

    def close(self) -> None:
        if self.handle:
            self.dev.lib.opevo_kernel_release(self.handle)
            self.handle = None

    def run(self) -> None:
        err = _errbuf()
        _check(self.dev.lib.opevo_kernel_run(self.handle, err, len(err)), err)

    def check(self, tol: float = 1e-2) -> float:
        rel = C.c_double()
        err = _errbuf()
        _check(self.dev.lib.opevo_kernel_check(self.handle, tol, C.byref(rel), err, len(err)), err)
        return rel.value

    def trace(self, ctas: int, launches: int = 1):
        """Phase stamps of `launches` back-to-back launches (instance built with
        -DOPEVO_TRACE=1): array [launches][ctas][16] (squeezed for one launch)."""
        import numpy as np

        out = np.zeros(launches * ctas * 16, dtype=np.uint64)
        err = _errbuf()
        _check(self.dev.lib.opevo_kernel_trace(
            self.handle, out.ctypes.data_as(C.POINTER(C.c_uint64)), out.size, err, len(err)), err)
        out = out.reshape(launches, ctas, 16)
        return out[0] if launches == 1 else out

    def time(self, warmup: int = 3, reps: int = 20, flush_l2: bool = False) -> float:
        ms = C.c_double()
        err = _errbuf()
        _check(self.dev.lib.opevo_kernel_time(self.handle, warmup, reps, int(flush_l2),
                                              C.byref(ms), err, len(err)), err)
        return ms.value


def time_rotating(kernels: "list[Kernel]", warmup: int = 1, reps: int = 64) -> float:
    """ms per launch of `reps` back-to-back launches cycling through kernels
    of one instance bound to distinct operand copies (HBM-fed steady state;
    ``opevo_kernels_time_rotating``)."""
    if not kernels:
        raise ValueError("no kernels")
    arr = (C.c_void_p * len(kernels))(*[k.handle for k in kernels])
    ms = C.c_double()
    err = _errbuf()
    lib = kernels[0].dev.lib
    _check(lib.opevo_kernels_time_rotating(arr, len(kernels), warmup, reps, C.byref(ms), err, len(err)), err)
    return ms.value


class PinnedBuffer:
    """Page-locked host memory from the driver (for honest H2D/D2H timing)."""

    def __init__(self, nbytes: int):
        self.lib = load()
        self.ptr = self.lib.opevo_host_alloc(nbytes)
        if not self.ptr:
            raise OpevoError(ERR_NO_DEVICE, "cuMemAllocHost failed (create a Device first)")
        self.nbytes = nbytes

    def array(self, dtype):
        import numpy as np

        buf = (C.c_char * self.nbytes).from_address(self.ptr)
        return np.frombuffer(buf, dtype=dtype)

    def close(self) -> None:
        if self.ptr:
            self.lib.opevo_host_free(self.ptr)
            self.ptr = None
