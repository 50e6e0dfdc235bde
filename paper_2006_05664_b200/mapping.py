"""OpEvo configuration -> sm_100a kernel knobs.

The paper's MatMul space (reference ``benchmarks.py:113-146``)
factors each output dimension into four levels -- blocks, virtual threads,
threads per block, per-thread tile -- and K into (outer, shared, inner).  On
Blackwell one thread issues each tensor-core MMA and the accumulator lives in
TMEM, so the levels map as:

=====================  ==============================================================
configuration          B200 kernel knob
=====================  ==============================================================
``n[0]``, ``m[0]``     CTA grid; CTA tile ``BM = N / n[0]``, ``BN = M / m[0]``
                       (UMMA shape: BM in {128, 256 = two M=128 atoms},
                       BN multiple of 16 in [16, 256])
``m[1]``               with OPEVO_MAP_MULTICAST=1 only: CTAs of a cluster along the
                       column-tile axis that share one TMA-multicast A tile,
                       ``cluster = largest c in {4, 2, 1} dividing m[1] and m[0]``;
                       by default canonicalised away like ``n[2..3]`` (see
                       ``_multicast_enabled``)
``n[1..3]``, ``m[2..3]`` the warp/thread split of the CTA tile: no tcgen05 counterpart
                       (canonicalised away -- many configurations, one kernel)
``k[0]``               split-K factor (CTAs along K, in-kernel deterministic reduce)
``k[2]``               BK: K elements per TMA stage (16, 32 or a multiple of 64)
``k[1]``               K blocks per CTA = K / (k[0] * k[2]) (derived)
``stages`` (added)     TMA->MMA ring depth, clamped to what fits in 227 KB
=====================  ==============================================================

Conv2d (``conv2d_space``) is an implicit GEMM over NHWC:
rows = output pixels, cols = Cout, K = (kh, kw, Cin).  ``co[0]`` -> BN =
Cout / co[0]; ``ho[0]``, ``wo[0]`` -> the output tile TILE_H = Ho / ho[0],
TILE_W = Wo / wo[0] (BM = 128 pixels = TILE_N x TILE_H x TILE_W); ``ci[0]`` ->
BK = Cin / ci[0] channels per stage; ``kh[0] * kw[0]`` -> split-K over filter
taps; ``unroll_step`` -> pipeline stages {0:2, 16:3, 64:4, 512:6, 1500:8};
``unroll_explicit`` = on selects the weight-resident variant when it applies
(BN = Cout, BK a multiple of 64, no split over taps): the whole BN x K weight
panel is loaded once per CTA and stays in shared memory -- the K loop is
"unrolled" over resident weights -- so the stages carry activations only.

A configuration whose mapping is infeasible is *invalid* and scores 0, as an
un-compilable TVM configuration does in the paper.
"""

from __future__ import annotations

from dataclasses import dataclass

from .operators import (
    UNROLL_ON,
    BatchMatMulSpec,
    Conv2dSpec,
    MatMulSpec,
    OperatorSpec,
    batchmatmul_space,
    conv2d_space,
    matmul_space,
)
from .spaces import Discrete, SearchSpace

SMEM_LIMIT = 232448          # 227 KB opt-in per CTA on B200
B200_SMS = 148
MAX_SPLIT = 16               # OPEVO_MAX_SPLIT: split-K workspace slices allocated at prepare
SMEM_EXTRA = 1024 + 256      # alignment slack + barriers
SM_SMEM_BYTES = 233472       # B200 shared memory per SM
CTA_RESERVED_SMEM = 1024     # reserved per resident CTA
STAGE_VALUES = (2, 3, 4, 5, 6, 7, 8)
UNROLL_TO_STAGES = {0: 2, 16: 3, 64: 4, 512: 6, 1500: 8}

FAMILY_GEMM = 0
FAMILY_CONV = 1
FAMILY_SIMT = 2            # fp32 MatMul: the paper's TVM dense schedule on CUDA cores
FAMILY_TF32X3 = 3          # fp32 MatMul / BMM on tcgen05: three kind::tf32 MMAs per K step


@dataclass(frozen=True)
class Knobs:
    """Canonical kernel knobs (order = ``opevo_knob`` in include/opevo.h)."""

    bm: int
    bn: int
    bk: int
    stages: int
    split: int = 1
    cluster: int = 1
    tile_h: int = 1
    tile_w: int = 1
    acc: int = 1
    cta_group: int = 1
    grid: int = 0
    b_res: int = 0           # conv: weight panel resident in shared memory
    bpu: int = 1             # BatchMatMul: batches per work unit
    line: int = 0            # conv: padded lines of 16 / 32 tile rows (0: dense tile / halo)
    panel_bytes: int = 0     # size of the resident panel (BN x K x 2; not a code knob)
    family: int = 0          # kernel family / batched operator (set by the mapping; decide
    batched: int = 0         # which split-K reduction is compiled in)

    def as_tuple(self) -> tuple[int, ...]:
        return (self.bm, self.bn, self.bk, self.stages, self.split, self.cluster,
                self.tile_h, self.tile_w, self.acc, self.cta_group, self.grid, self.b_res, self.bpu,
                self.line)

    def tma_split(self) -> int:
        """Split factor compiled in when the K slices reduce through fp32
        partials moved by TMA in one wave (mirrors ``tma_split`` in
        csrc/opevo.cpp), else 0."""
        s = self.split
        ok = (self.family == FAMILY_GEMM and not self.batched and s in (2, 4) and self.cta_group == 1
              and self.cluster == 1 and self.bm == 128 and self.acc == 1 and self.bpu <= 1
              and self.bn % 32 == 0 and (s - 1) * 128 * self.bn * 4 <= 196608)
        return s if ok else 0

    def dsmem_split(self) -> int:
        """Split factor compiled in when the K slices reduce through DSMEM
        (mirrors ``dsmem_split`` in csrc/opevo.cpp), else 0."""
        s = self.split
        ld = self.bn + 4
        red = self.bm * ld * 4 + (s - 1) * (self.bm // max(s, 1)) * ld * 4
        ok = (s in (2, 4, 8) and self.cta_group == 1 and self.cluster == 1 and self.bm == 128
              and not self.tma_split() and not (self.family == FAMILY_CONV and self.line)
              and _align1k(red) + epi_bytes(self.bn, self.family == FAMILY_TF32X3) + SMEM_EXTRA
              <= SMEM_LIMIT)
        return s if ok else 0

    def halo_kw(self) -> int:
        """Conv "halo lines" (mirrors ``halo_kw`` in csrc/opevo.cpp): a tile
        width that does not divide BM marks lines of 17 - KW pixels padded to
        16 rows, one TMA box per filter row; returns KW, else 0."""
        if (self.family == FAMILY_CONV and self.line == 0 and 1 <= self.tile_w < 16 and self.tile_h >= 1
                and self.bm_cta % (self.tile_h * self.tile_w)):
            return 17 - self.tile_w
        return 0

    @property
    def bm_cta(self) -> int:
        """Tile rows one CTA holds (a CTA pair splits BM = 256 in two)."""
        return self.bm // 2 if self.cta_group == 2 else self.bm

    def compile_key(self) -> tuple[int, ...]:
        """Fields that change the generated code (split-K is a launch arg
        except for DSMEM-reduced splits)."""
        return (self.bm, self.bn, self.bk, self.stages, self.cluster, self.tile_h, self.tile_w,
                self.acc, self.cta_group, self.dsmem_split(), self.tma_split(), self.b_res, self.bpu,
                self.line)

    def narrow_epi(self) -> bool:
        """Two-CTAs-per-SM rule (mirrors ``narrow_epi`` in csrc/opevo.cpp): a
        single-CTA or CTA-pair bf16 instance that fits twice on an SM only with 32-column
        epilogue staging (16 KB instead of 32 KB) uses it."""
        if (self.family not in (FAMILY_GEMM, FAMILY_CONV) or self.bn % 64 or self.acc != 1
                or self.cluster != 1 or self.dsmem_split() or self.b_res or self.tmem_alloc_cols() > 256):
            return False
        base = self._pipe_bytes() + SMEM_EXTRA + CTA_RESERVED_SMEM
        return 2 * (base + epi_bytes(64)) > SM_SMEM_BYTES and 2 * (base + epi_bytes(32)) <= SM_SMEM_BYTES

    def tmem_alloc_cols(self) -> int:
        """TMEM columns the kernel allocates (mirrors ``tmem_alloc_cols`` in
        csrc/opevo.cpp: four accumulator buffers when they fit in half of
        TMEM, else two, else one; rounded up to a power of two >= 32)."""
        used = (2 if self.bm_cta == 256 else 1) * self.bn * self.acc * max(1, self.bpu)
        want = (4 if 4 * used <= 256 else 2 if 2 * used <= 512 else 1) * used
        cols = 32
        while cols < want:
            cols *= 2
        return cols

    def _epi(self) -> int:
        return epi_bytes(32 if self.narrow_epi() else self.bn)

    def _pipe_bytes(self) -> int:
        if self.halo_kw():
            return _align1k((self.bm_cta + self.halo_kw() * self.bn // self.cta_group) * self.bk * 2 * self.stages)
        x3 = self.family == FAMILY_TF32X3
        if x3:   # fp32 operands (bf16 pairs) staged twice: hi as landed + lo
            pipe = 2 * stage_bytes(self.bm, self.bn, 2 * self.bk) * self.stages
        else:
            pipe = stage_bytes(self.bm, self.bn, self.bk, self.cta_group) * self.stages * self.bpu
        if self.dsmem_split():
            ld = self.bn + 4
            pipe = max(pipe, self.bm * ld * 4 + (self.split - 1) * (self.bm // self.split) * ld * 4)
        if self.tma_split():
            pipe = max(pipe, max(self.split - 1, 1) * 128 * self.bn * 4)
        return _align1k(pipe)

    def smem_bytes(self) -> int:
        """Mirrors ``smem_bytes`` in csrc/opevo.cpp (bf16 output)."""
        if self.b_res:
            return _align1k(self.bm * self.bk * 2 * self.stages) + epi_bytes(self.bn) + 2048 + self.panel_bytes
        x3 = self.family == FAMILY_TF32X3
        return self._pipe_bytes() + (epi_bytes(self.bn, True) if x3 else self._epi()) + SMEM_EXTRA


@dataclass(frozen=True)
class Mapped:
    """Result of mapping one configuration."""

    knobs: Knobs | None
    reason: str = ""
    family: int = FAMILY_GEMM
    batched: bool = False

    @property
    def valid(self) -> bool:
        return self.knobs is not None


def _align1k(n: int) -> int:
    return (n + 1023) // 1024 * 1024


def epi_bytes(bn: int, out_f32: bool = False) -> int:
    """TMA-store staging of the epilogue: 4 warps x 2 buffers x 32 rows x
    STORE_COLS (bf16 output: 64, 32 or 16, the widest dividing BN; fp32
    output: 32 or 16)."""
    if out_f32:
        return 4 * 2 * 32 * (32 if bn % 32 == 0 else 16) * 4
    return 4 * 2 * 32 * (64 if bn % 64 == 0 else 32 if bn % 32 == 0 else 16) * 2


def stage_bytes(bm: int, bn: int, bk: int, cta_group: int = 1) -> int:
    """Shared memory per pipeline stage of one CTA (a CTA pair stages BM/2 rows
    of A and BN/2 rows of B in each CTA)."""
    if cta_group == 2:
        return (bm // 2 + bn // 2) * bk * 2
    return (bm + bn) * bk * 2


def _bk_ok(bk: int) -> bool:
    return bk in (16, 32) or (64 <= bk <= 256 and bk % 64 == 0)


def _fit_stages(want: int, bm: int, bn: int, bk: int, cta_group: int = 1, bpu: int = 1,
                x3: bool = False) -> int:
    """Largest ring depth <= want whose shared memory (pipeline, epilogue
    staging, barriers) fits in 227 KB; 0 when not even one stage fits.
    ``x3``: 3xTF32 (fp32 BK, hi + lo areas per stage, fp32 output)."""
    sb = 2 * stage_bytes(bm, bn, 2 * bk) if x3 else stage_bytes(bm, bn, bk, cta_group) * bpu
    s = want
    while s > 0 and _align1k(s * sb) + epi_bytes(bn, x3) + SMEM_EXTRA > SMEM_LIMIT:
        s -= 1
    return s


def _multicast_enabled() -> bool:
    """``m[1]`` -> A-multicast cluster only with OPEVO_MAP_MULTICAST=1.  Off by
    default: multicast never won on any BASELINE operator (cluster <= 4
    unicast loads of one tile are deduplicated in L2 anyway), and the extra
    instance per ``m[1]`` parity made the landscape rugged -- at 1024^3, 6 of
    8 seeds reached the best instance with it, 8 of 8 without
    (profiles/round2/seeds/).  The library keeps the knob."""
    import os

    return os.environ.get("OPEVO_MAP_MULTICAST", "0") == "1"


def _largest_pow2_divisor(*vals: int, cap: int = 4) -> int:
    c = cap
    while c > 1 and any(v % c for v in vals):
        c //= 2
    return c


def gpu_operator_space(spec: OperatorSpec, dtype: str = "bf16") -> SearchSpace:
    """The reference space of ``spec`` plus the B200-only knob(s), declared in
    the reference's JSON space format (so the reference engine can replay a
    B200 trajectory).  fp32 MatMul uses the reference space unchanged: every
    factor is a knob of the SIMT family."""
    if dtype == "f32":
        if not isinstance(spec, (MatMulSpec, BatchMatMulSpec)):
            raise TypeError("fp32 is served for MatMul / BatchMatMul only")
        return matmul_space(spec) if isinstance(spec, MatMulSpec) else batchmatmul_space(spec)
    if dtype == "tf32x3" and not isinstance(spec, (MatMulSpec, BatchMatMulSpec)):
        raise TypeError("3xTF32 is served for MatMul / BatchMatMul only")
    if isinstance(spec, MatMulSpec):
        base = matmul_space(spec)
    elif isinstance(spec, BatchMatMulSpec):
        base = batchmatmul_space(spec)
    elif isinstance(spec, Conv2dSpec):
        return conv2d_space(spec)
    else:
        raise TypeError(f"unknown operator spec: {spec!r}")
    return SearchSpace(list(zip(base.names, base.spaces)) + [("stages", Discrete(STAGE_VALUES))])


def _gemm_knobs(rows: int, cols: int, depth: int, vals: dict,
                batch: int = 0) -> tuple[Knobs | None, str]:
    n, m, k = vals["n"], vals["m"], vals["k"]
    bm, bn = rows // n[0], cols // m[0]
    split, bk = k[0], k[2]
    if bm not in (128, 256):
        return None, f"BM={bm} is not a UMMA row tile (128 or 256)"
    if split > MAX_SPLIT:
        return None, f"split-K {split} exceeds the {MAX_SPLIT}-slice workspace"
    if bn % 16 or not 16 <= bn <= 256:
        return None, f"BN={bn} is not a UMMA column tile (16..256, step 16)"
    if not _bk_ok(bk):
        return None, f"BK={bk} is not a TMA/UMMA K stage (16, 32, 64k)"
    # a 256-row tile with an even row vthread split runs on a CTA pair
    # (cta_group::2): the pair's two SMs each hold 128 rows
    cta_group = 2 if (bm == 256 and n[1] % 2 == 0) else 1
    if (2 if (bm == 256 and cta_group == 1) else 1) * bn > 512:
        return None, "accumulator exceeds TMEM"
    bpu = _batches_per_unit(vals, batch, bm, bn, bk, split, cta_group)
    stages = _fit_stages(int(vals.get("stages", 4)), bm, bn, bk, cta_group, bpu)
    if stages < 1:
        return None, "one stage does not fit in shared memory"
    cluster = (1 if (cta_group == 2 or bpu > 1 or not _multicast_enabled())
               else _largest_pow2_divisor(m[1], m[0]))
    kn = Knobs(bm, bn, bk, stages, split, cluster, cta_group=cta_group, bpu=bpu,
               batched=int(bool(batch)))
    if kn.tma_split() and (rows // bm) * (cols // bn) * split > B200_SMS:
        # slice 0 of a tile waits for the others: every slice must be resident
        return None, "TMA split-K needs one wave of CTAs"
    return kn, ""


def _x3_knobs(rows: int, cols: int, vals: dict, batch: int = 0) -> tuple[Knobs | None, str]:
    """3xTF32 family: the bf16 GEMM mapping with BK = k[2] fp32 elements (a
    stage of 2*BK bf16-unit bytes per row, landed once and split into hi and
    lo areas), single-CTA tiles (BM 256 = two M=128 atoms), no multicast."""
    n, m, k = vals["n"], vals["m"], vals["k"]
    bm, bn = rows // n[0], cols // m[0]
    split, bk = k[0], k[2]
    if bm not in (128, 256):
        return None, f"BM={bm} is not a UMMA row tile (128 or 256)"
    if split > MAX_SPLIT:
        return None, f"split-K {split} exceeds the {MAX_SPLIT}-slice workspace"
    if bn % 16 or not 16 <= bn <= 256:
        return None, f"BN={bn} is not a UMMA column tile (16..256, step 16)"
    if not _bk_ok(2 * bk):
        return None, f"BK={bk} fp32 is not a TMA/UMMA K stage (8, 16, 32k)"
    if (2 if bm == 256 else 1) * bn > 512:
        return None, "accumulator exceeds TMEM"
    stages = _fit_stages(int(vals.get("stages", 4)), bm, bn, bk, x3=True)
    if stages < 1:
        return None, "one stage does not fit in shared memory"
    return Knobs(bm, bn, bk, stages, split, 1, family=FAMILY_TF32X3, batched=int(bool(batch))), ""


def _batches_per_unit(vals: dict, batch: int, bm: int, bn: int, bk: int, split: int,
                      cta_group: int) -> int:
    """BatchMatMul: the batch factor's inner level ``b[1]`` (batches handled by
    one block in the paper's schedule) -> consecutive batches per CTA work
    unit, the largest of {4, 2, 1} dividing it: one TMA box per operand and
    stage then carries all of them (a box costs about the same whatever its
    size) and their accumulators sit side by side in TMEM.  Single-CTA
    128-row tiles without a K split only (mirrors ``bpu`` in csrc/opevo.cpp)."""
    if not batch or "b" not in vals or bm != 128 or cta_group != 1 or split != 1:
        return 1
    if bk > 32 and bk % 64:
        return 1
    u = _largest_pow2_divisor(vals["b"][1], batch)
    while u > 1 and 2 * u * bn > 512:        # two TMEM buffers of u x BN columns
        u //= 2
    return u


def conv_channels_padded(cin: int) -> int:
    """Cin in the conv kernels' layout: padded with zeros to a multiple of 16
    (a pixel row must be >= 16 bytes for TMA and hold whole 32-byte UMMA K
    steps; AlexNet conv1's Cin = 3 -> 16).  Mirrors op->cpad in csrc/opevo.cpp."""
    return (cin + 15) // 16 * 16


def _conv_knobs(spec: Conv2dSpec, vals: dict) -> tuple[Knobs | None, str]:
    co, ho, wo, ci = vals["co"], vals["ho"], vals["wo"], vals["ci"]
    kh, kw = vals["kh"], vals["kw"]
    s_ = spec.stride
    bn = spec.out_channels // co[0]
    th, tw = spec.out_height // ho[0], spec.out_width // wo[0]
    cpad = conv_channels_padded(spec.in_channels)
    if cpad % ci[0]:
        return None, f"BK = {cpad} padded channels / {ci[0]} is not whole"
    bk = cpad // ci[0]
    # an even Cout virtual-thread split runs 256-pixel tiles (each tap's
    # activation box twice as large; a TMA box costs about the same whatever
    # its size, so this halves the boxes): two M=128 atoms in one CTA, or --
    # with an even H virtual-thread split -- a CTA pair (cta_group::2, each
    # SM holds 128 pixel rows and half the weight tile)
    bm = 256 if co[1] % 2 == 0 else 128
    cg = 2 if (bm == 256 and ho[1] % 2 == 0) else 1
    # a Cout split by four on a CTA pair of halo lines: 256 rows per CTA (two
    # M=256 atoms per K step, one 32 KB activation box per filter row)
    if (cg == 2 and co[1] % 4 == 0 and s_ == 1 and tw + spec.kernel_w - 1 == 16
            and kh[0] * kw[0] == 1 and (cpad // ci[0]) % 64 == 0):
        bm = 512
    bm_cta = bm // 2 if cg == 2 else bm
    if bn % 16 or not 16 <= bn <= 256:
        return None, f"BN={bn} is not a UMMA column tile"
    if bm == 256 and cg == 1 and 2 * bn > 512:
        return None, "accumulator exceeds TMEM"
    if not _bk_ok(bk):
        return None, f"BK={bk} channels is not a TMA/UMMA K stage"
    if s_ == 1 and tw + spec.kernel_w - 1 == 16 and bm_cta % (th * tw):
        return _conv_halo_knobs(spec, vals, bm, bn, bk, th, tw, cg)
    split = kh[0] * kw[0]
    line = 0
    if split > MAX_SPLIT:
        return None, f"split over {split} filter taps exceeds the {MAX_SPLIT}-slice workspace"
    if th * tw > bm_cta or bm_cta % (th * tw):
        # padded lines: TILE_W <= LINE output pixels per line of LINE rows
        # (TILE_N = floor(rows / (LINE x TILE_H)) images; rows past them are junk)
        line = 16 if tw <= 16 else 32 if tw <= 32 else 0
        if not line or line * th > bm_cta:
            return None, f"output tile {th}x{tw} neither divides {bm_cta} pixels nor packs in lines"
        tn = bm_cta // (line * th)
        rows_w = line
    else:
        tn = bm_cta // (th * tw)
        rows_w = tw
    if spec.batch % (tn * cg) or tn > 256 or th > 256 or tw > 256:
        return None, f"image tile {tn * cg} does not divide the batch {spec.batch}"
    if rows_w * s_ > 256 or th * s_ > 256:
        return None, f"stride {s_}: the activation box would exceed 256 pixels"
    want = UNROLL_TO_STAGES[vals["unroll_step"]]
    if vals.get("unroll_explicit") == UNROLL_ON and cg == 1:
        stages, panel = _conv_resident_fit(spec, bn, bk, split, want, bm)
        if stages:
            return Knobs(bm, bn, bk, stages, split, 1, th, tw, b_res=1, panel_bytes=panel, line=line,
                         family=FAMILY_CONV), ""
    stages = _fit_stages(want, bm, bn, bk, cg)
    if stages < 1:
        return None, "one stage does not fit in shared memory"
    return Knobs(bm, bn, bk, stages, split, 1, th, tw, cta_group=cg, line=line, family=FAMILY_CONV), ""


def _conv_halo_knobs(spec: Conv2dSpec, vals: dict, bm: int, bn: int, bk: int, th: int,
                     tw: int, cg: int = 1) -> tuple[Knobs | None, str]:
    """Halo lines: output lines of TILE_W = 17 - KW pixels, each padded to 16
    tile rows, so one TMA box {Cin block, 16, TILE_H, TILE_N} per filter row
    serves all KW taps of that row (mirrors OPEVO_HALO in gemm_sm100.cuh).
    On a CTA pair each CTA holds TILE_N of the pair's 2 x TILE_N images."""
    kh, kw = vals["kh"], vals["kw"]
    bm_cta = bm // 2 if cg == 2 else bm
    if bm_cta % (16 * th):
        return None, f"{bm_cta} rows do not hold 16-row lines x {th} rows"
    tn = bm_cta // (16 * th)
    if spec.batch % (tn * cg) or spec.padding >= spec.kernel_w:
        return None, f"image tile {tn * cg} does not divide the batch {spec.batch}"
    if bk % 64 or kh[0] * kw[0] != 1:
        return None, "halo lines need BK a multiple of 64 and no split over taps"
    want = UNROLL_TO_STAGES[vals["unroll_step"]]
    if vals.get("unroll_explicit") == UNROLL_ON and cg == 1:
        stages, panel = _conv_resident_fit(spec, bn, bk, 1, want, bm)
        if stages:
            return Knobs(bm, bn, bk, stages, 1, 1, th, tw, b_res=1, panel_bytes=panel,
                         family=FAMILY_CONV), ""
    stages = _fit_halo_stages(want, bm, bn, bk, spec.kernel_w, cg)
    if stages < 1:
        return None, "one stage does not fit in shared memory"
    return Knobs(bm, bn, bk, stages, 1, 1, th, tw, cta_group=cg, family=FAMILY_CONV), ""


def _fit_halo_stages(want: int, bm: int, bn: int, bk: int, kw: int, cg: int = 1) -> int:
    """Stages of a streaming halo-lines conv: each holds the activation box
    and the KW weight tiles of one filter row (a CTA pair: 128 rows and half
    of each weight tile per CTA)."""
    rows = (bm // 2 if cg == 2 else bm) + kw * bn // cg
    s = want
    while s > 0 and _align1k(s * rows * bk * 2) + epi_bytes(bn) + SMEM_EXTRA > SMEM_LIMIT:
        s -= 1
    return s


def _conv_resident_fit(spec: Conv2dSpec, bn: int, bk: int, split: int, want: int,
                       bm: int = 128) -> tuple[int, int]:
    """(stages, panel bytes) of the weight-resident conv variant -- the whole
    BN x K weight panel loaded once per CTA, stages carry activations only --
    or (0, 0) when it does not apply (needs BN = Cout, BK a multiple of 64, no
    split over taps, the panel plus two stages within 227 KB).  Mirrors
    ``b_resident`` / the panel check in csrc/opevo.cpp."""
    depth = spec.kernel_h * spec.kernel_w * conv_channels_padded(spec.in_channels)
    if bn != spec.out_channels or bk % 64 or split != 1 or depth // 64 > 256:
        return 0, 0
    panel = bn * depth * 2
    s = want
    while s > 0 and _align1k(s * bm * bk * 2) + epi_bytes(bn) + 2048 + panel > SMEM_LIMIT:
        s -= 1
    return (s, panel) if s >= 2 else (0, 0)


def _simt_knobs(vals: dict) -> tuple[Knobs | None, str]:
    """fp32 SIMT family: the paper's levels map one to one (knob slots 0..7 =
    n2, n3, n4, m2, m3, m4, k2, k3; n1, m1 follow from the shape, k1 = K/(k2 k3))."""
    n, m, k = vals["n"], vals["m"], vals["k"]
    threads = n[2] * m[2]
    if threads > 1024:
        return None, f"n3*m3 = {threads} threads per block exceeds 1024"
    if n[1] * n[3] * m[1] * m[3] > 256:
        return None, "per-thread tile exceeds the register file"
    ks = k[1] * k[2]
    smem = ks * (n[1] * n[2] * n[3] + m[1] * m[2] * m[3] + 2) * 4
    if k[2] > 64 or smem > SMEM_LIMIT:
        return None, f"shared tile {smem} B (k3={k[2]}) too large"
    return Knobs(n[1], n[2], n[3], m[1], m[2], m[3], k[1], k[2]), ""


def config_to_knobs(spec: OperatorSpec, space: SearchSpace, config: tuple,
                    dtype: str = "bf16") -> Mapped:
    """Map one configuration of ``space`` to kernel knobs (or an invalid reason)."""
    vals = dict(zip(space.names, config))
    if dtype == "f32":
        kn, why = _simt_knobs(vals)
        return Mapped(kn, why, FAMILY_SIMT, isinstance(spec, BatchMatMulSpec))
    if dtype == "tf32x3":
        if isinstance(spec, MatMulSpec):
            kn, why = _x3_knobs(spec.n, spec.m, vals)
            return Mapped(kn, why, FAMILY_TF32X3, False)
        if isinstance(spec, BatchMatMulSpec):
            kn, why = _x3_knobs(spec.n, spec.m, vals, batch=spec.b)
            return Mapped(kn, why, FAMILY_TF32X3, True)
        raise TypeError("3xTF32 is served for MatMul / BatchMatMul only")
    if isinstance(spec, MatMulSpec):
        kn, why = _gemm_knobs(spec.n, spec.m, spec.k, vals)
        return Mapped(kn, why, FAMILY_GEMM, False)
    if isinstance(spec, BatchMatMulSpec):
        kn, why = _gemm_knobs(spec.n, spec.m, spec.k, vals, batch=spec.b)
        return Mapped(kn, why, FAMILY_GEMM, True)
    if isinstance(spec, Conv2dSpec):
        kn, why = _conv_knobs(spec, vals)
        return Mapped(kn, why, FAMILY_CONV, False)
    raise TypeError(f"unknown operator spec: {spec!r}")


def valid_fraction(spec: OperatorSpec, space: SearchSpace, samples: int = 20000,
                   seed: int = 0, dtype: str = "bf16") -> float:
    """Monte-Carlo fraction of uniformly drawn configurations that map."""
    import numpy as np

    rng = np.random.default_rng(seed)
    ok = sum(config_to_knobs(spec, space, space.sample_uniform(rng), dtype).valid
             for _ in range(samples))
    return ok / samples
