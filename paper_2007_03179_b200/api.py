"""Host-side mirror of the reference's SpMM-like interface, over the C ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/spmm/), so the parity tests read like the
reference's own tests:

  CsrMatrix, from_coo                csr.hpp:22-35, 58-93
  DenseMatrix, make_random_dense,    dense.hpp:14-38, 51-59, 62-72
    checksum
  ReduceOp, ops.sum/max (+mean/min), reduce_op.hpp:14-36
    reduce_op_by_name
  KernelVariant, variant_by_name,    kernel.hpp:44-98
    select_variant, check_config
  FaultMode, ExecOptions             kernel.hpp:167-186
  native_spmm, bench                 native.hpp:101-180
  GraphGenSpec, gen_uniform_random,  generate.hpp:14-80
    randomize_values
  save_csr_cache, read_csr_cache,    io.hpp:50-115 (CSR1 binary cache)
    load_matrix, DeviceCsr.load

Compute goes through libgespmm.so only (CUDA, sm_100a); ``workers`` is
accepted for signature compatibility and ignored.  Two device-level entry
points are added for callers that keep data in HBM: :func:`spmm` (torch
tensors) and :class:`Plan` (inspect once, execute many).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import time
from typing import List, Optional, Tuple

import numpy as np

from . import _lib
from ._lib import Csr, default_options, lib


class Error(RuntimeError):
    """spmm::Error (common.hpp:17-21); ``status`` is the C-ABI status code."""

    def __init__(self, what: str, status: int = _lib.EINVAL):
        super().__init__(what)
        self.status = status


def _check(status: int):
    if status != _lib.OK:
        raise Error(_lib.last_error(), status)


# ---------------------------------------------------------------------------
# data model
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class CsrMatrix:
    """Canonical CSR (csr.hpp:22-35): u32 row_ptr[n_rows+1], u32 col_ind[nnz], f32 vals[nnz]."""
    n_rows: int = 0
    n_cols: int = 0
    row_ptr: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(1, np.uint32))
    col_ind: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.uint32))
    vals: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.float32))

    @classmethod
    def empty(cls, rows: int, cols: int) -> "CsrMatrix":
        return cls(rows, cols, np.zeros(rows + 1, np.uint32), np.zeros(0, np.uint32),
                   np.zeros(0, np.float32))

    def nnz(self) -> int:
        return int(len(self.col_ind))

    def row_len(self, r: int) -> int:
        return int(self.row_ptr[r + 1]) - int(self.row_ptr[r])

    def mean_degree(self) -> float:
        return 0.0 if self.n_rows == 0 else self.nnz() / self.n_rows

    def _c(self) -> Tuple[Csr, tuple]:
        rp = np.ascontiguousarray(self.row_ptr, np.uint32)
        ci = np.ascontiguousarray(self.col_ind, np.uint32)
        v = np.ascontiguousarray(self.vals, np.float32)
        s = Csr(self.n_rows, self.n_cols, len(ci), rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
        return s, (rp, ci, v)


@dataclasses.dataclass
class DenseMatrix:
    """Row-major f32 (dense.hpp:14-38)."""
    n_rows: int = 0
    n_cols: int = 0
    data: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros((0, 0), np.float32))
    base_alignment: int = 128

    @classmethod
    def zeros(cls, rows: int, cols: int, fill: float = 0.0) -> "DenseMatrix":
        return cls(rows, cols, np.full((rows, cols), fill, np.float32))

    @classmethod
    def of(cls, arr) -> "DenseMatrix":
        a = np.ascontiguousarray(arr, np.float32)
        return cls(a.shape[0], a.shape[1], a)

    def at(self, r: int, c: int) -> float:
        return float(self.data[r, c])

    def size(self) -> int:
        return self.n_rows * self.n_cols

    def same_shape(self, o: "DenseMatrix") -> bool:
        return self.n_rows == o.n_rows and self.n_cols == o.n_cols

    def bitwise_equal(self, o: "DenseMatrix") -> bool:
        return self.same_shape(o) and np.array_equal(
            np.ascontiguousarray(self.data, np.float32).view(np.uint32),
            np.ascontiguousarray(o.data, np.float32).view(np.uint32))


def check_dense_valid(m: DenseMatrix):
    """dense.hpp:40-46."""
    if m.data.size != m.n_rows * m.n_cols:
        raise Error("dense matrix: data length does not match n_rows * n_cols")
    ba = m.base_alignment
    if ba == 0 or (ba & (ba - 1)) != 0 or ba > 4096:
        raise Error("dense matrix: base_alignment must be a power of two <= 4096")


def from_coo(n_rows: int, n_cols: int, entries, policy: str = "sum") -> CsrMatrix:
    """COO triples -> canonical CSR (csr.hpp:58-93) through gespmm_from_coo:
    ordered by (row, col), duplicates collapse in input order by policy
    ``sum`` or ``last``."""
    if policy not in ("sum", "last"):
        raise Error(f"from_coo: unknown dedup policy '{policy}' (sum, last)")
    if isinstance(entries, tuple) and len(entries) == 3 and hasattr(entries[0], "__len__") \
            and not np.isscalar(entries[0]):
        rows, cols, vals = entries
    else:
        ent = list(entries)
        rows = [e[0] for e in ent]
        cols = [e[1] for e in ent]
        vals = [e[2] for e in ent]
    r = np.asarray(rows, np.int64)
    c = np.asarray(cols, np.int64)
    if r.size and (r.min() < 0 or c.min() < 0 or r.max() > 0xffffffff or c.max() > 0xffffffff):
        i = int(np.nonzero((r < 0) | (c < 0) | (r > 0xffffffff) | (c > 0xffffffff))[0][0])
        raise Error(f"coo entry ({r[i]}, {c[i]}, {float(np.float32(vals[i])):g}) outside declared "
                    f"{n_rows}x{n_cols} bounds")
    r = np.ascontiguousarray(r, np.uint32)
    c = np.ascontiguousarray(c, np.uint32)
    v = np.ascontiguousarray(vals, np.float32)
    cnt = len(r)
    rp = np.zeros(n_rows + 1, np.uint32)
    ci = np.empty(max(cnt, 1), np.uint32)
    vv = np.empty(max(cnt, 1), np.float32)
    nnz = C.c_uint64()
    _check(lib().gespmm_from_coo(n_rows, n_cols, cnt, r.ctypes.data if cnt else None,
                                 c.ctypes.data if cnt else None, v.ctypes.data if cnt else None,
                                 0 if policy == "sum" else 1, rp.ctypes.data, ci.ctypes.data,
                                 vv.ctypes.data, C.byref(nnz)))
    z = nnz.value
    return CsrMatrix(n_rows, n_cols, rp, ci[:z].copy(), vv[:z].copy())


def to_coo(m: CsrMatrix):
    """CSR -> (n_rows, n_cols, [(row, col, val), ...]) in row-major order (csr.hpp:95-104)."""
    rows = np.repeat(np.arange(m.n_rows, dtype=np.uint32), np.diff(m.row_ptr.astype(np.int64)))
    return m.n_rows, m.n_cols, list(zip(rows.tolist(), m.col_ind.tolist(),
                                        m.vals.astype(np.float32).tolist()))


@dataclasses.dataclass
class ValidationReport:
    """csr.hpp:107-110: one message per violation, empty iff canonical."""
    violations: List[str]

    def ok(self) -> bool:
        return not self.violations


def validate(m: CsrMatrix) -> ValidationReport:
    """Every canonical-CSR violation, in the reference's order and wording
    (csr.hpp:112-153), through gespmm_validate_host."""
    rp = np.ascontiguousarray(m.row_ptr, np.uint32)
    ci = np.ascontiguousarray(m.col_ind, np.uint32)
    s = Csr(m.n_rows, m.n_cols, len(ci), rp.ctypes.data if rp.size else None,
            ci.ctypes.data if ci.size else None, None)
    need = C.c_uint64()
    n = lib().gespmm_validate_host(C.byref(s), rp.size, ci.size, len(m.vals), None, 0,
                                   C.byref(need))
    if n == 0:
        return ValidationReport([])
    buf = C.create_string_buffer(need.value)
    lib().gespmm_validate_host(C.byref(s), rp.size, ci.size, len(m.vals), buf, need.value,
                               C.byref(need))
    return ValidationReport(buf.value.decode().split("\n"))


def require_canonical(m: CsrMatrix, who: str) -> None:
    """csr.hpp:155-158."""
    rep = validate(m)
    if not rep.ok():
        raise Error(f"{who}: matrix is not canonical CSR: {rep.violations[0]}", _lib.ENONCANON)


def parse_matrix_market(text) -> Tuple[int, int, list]:
    """matrix_market.hpp:60-160 (gespmm_mtx_parse): (n_rows, n_cols, triples)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    rows, cols, k = C.c_uint32(), C.c_uint32(), C.c_uint64()
    _check(lib().gespmm_mtx_parse(data, len(data), C.byref(rows), C.byref(cols), C.byref(k),
                                  None, None, None))
    r = np.empty(max(k.value, 1), np.uint32)
    c = np.empty(max(k.value, 1), np.uint32)
    v = np.empty(max(k.value, 1), np.float32)
    _check(lib().gespmm_mtx_parse(data, len(data), C.byref(rows), C.byref(cols), C.byref(k),
                                  r.ctypes.data, c.ctypes.data, v.ctypes.data))
    z = k.value
    return rows.value, cols.value, (r[:z], c[:z], v[:z])


# ---------------------------------------------------------------------------
# reduce ops and variants
# ---------------------------------------------------------------------------

_F32_MAX = float(np.finfo(np.float32).max)


@dataclasses.dataclass(frozen=True)
class ReduceOp:
    """reduce_op.hpp:14-20; the combine is fused into the kernel by name."""
    name: str
    init: float

    @property
    def code(self) -> int:
        return _lib.REDUCE[self.name]

    def fold(self, acc: float, x: float) -> float:
        """Host restatement of the combine, for documentation/tests of the laws."""
        a, b = np.float32(acc), np.float32(x)
        if self.name in ("sum", "mean"):
            return float(np.float32(a + b))
        if self.name == "max":
            return float(b if a < b else a)
        return float(b if b < a else a)


class ops:
    """ops::sum / ops::max (reduce_op.hpp:27-28) plus the new mean / min."""

    @staticmethod
    def sum() -> ReduceOp:
        return ReduceOp("sum", 0.0)

    @staticmethod
    def max() -> ReduceOp:
        return ReduceOp("max", -_F32_MAX)

    @staticmethod
    def mean() -> ReduceOp:
        return ReduceOp("mean", 0.0)

    @staticmethod
    def min() -> ReduceOp:
        return ReduceOp("min", _F32_MAX)


def reduce_op_by_name(name: str) -> ReduceOp:
    code = C.c_int()
    _check(lib().gespmm_reduce_by_name(name.encode(), C.byref(code)))
    return {0: ops.sum, 1: ops.mean, 2: ops.max, 3: ops.min}[code.value]()


class KernelKind(enum.IntEnum):
    Naive = _lib.VARIANT_NAIVE
    Crc = _lib.VARIANT_CRC
    CrcCwm = _lib.VARIANT_CRC_CWM
    Tuned = _lib.VARIANT_TUNED


@dataclasses.dataclass(frozen=True)
class KernelVariant:
    """kernel.hpp:48-68, plus ``tuned`` (the B200 design)."""
    kind: KernelKind = KernelKind.Naive
    cf: int = 1

    @staticmethod
    def naive() -> "KernelVariant":
        return KernelVariant(KernelKind.Naive, 1)

    @staticmethod
    def crc() -> "KernelVariant":
        return KernelVariant(KernelKind.Crc, 1)

    @staticmethod
    def crc_cwm(cf: int) -> "KernelVariant":
        return KernelVariant(KernelKind.CrcCwm, cf)

    @staticmethod
    def tuned() -> "KernelVariant":
        return KernelVariant(KernelKind.Tuned, 1)

    def cf_effective(self) -> int:
        return self.cf if self.kind == KernelKind.CrcCwm else 1

    def name(self) -> str:
        return {KernelKind.Naive: "naive", KernelKind.Crc: "crc", KernelKind.CrcCwm: "crc-cwm",
                KernelKind.Tuned: "tuned"}[self.kind]


def variant_by_name(name: str, cf: int = 2) -> KernelVariant:
    if name == "naive":
        return KernelVariant.naive()
    if name == "crc":
        return KernelVariant.crc()
    if name == "crc-cwm":
        return KernelVariant.crc_cwm(cf)
    if name == "tuned":
        return KernelVariant.tuned()
    raise Error(f"unknown kernel variant '{name}' (naive, crc, crc-cwm, tuned)")


def select_variant(n: int) -> KernelVariant:
    """The reference's dispatch rule (kernel.hpp:96-98), answered by the library."""
    v, cf = C.c_int32(), C.c_uint32()
    lib().gespmm_select_variant(n, C.byref(v), C.byref(cf))
    return KernelVariant(KernelKind(v.value), cf.value)


@dataclasses.dataclass(frozen=True)
class KernelConfig:
    warp_size: int = 32
    warps_per_block: int = 8
    variant: KernelVariant = KernelVariant.naive()


def check_config(cfg: KernelConfig):
    """kernel.hpp:83-92 (the device kernels always run warp_size 32)."""
    ws = cfg.warp_size
    if ws < 4 or ws > 64 or (ws & (ws - 1)) != 0:
        raise Error("warp_size must be a power of two in [4, 64]")
    if cfg.warps_per_block < 1:
        raise Error("warps_per_block must be >= 1")
    if cfg.variant.kind == KernelKind.CrcCwm and cfg.variant.cf not in (2, 4, 8):
        raise Error("coarsening factor must be 2, 4 or 8")


class FaultMode(enum.IntEnum):
    None_ = 0
    SkipTail = 1


@dataclasses.dataclass(frozen=True)
class ExecOptions:
    fault: FaultMode = FaultMode.None_
    exact: bool = True
    arg_kind: str = "edge"          # "edge" (CSR position p) or "column" (col_ind[p])
    l2_hints: int = 1               # 0 off; 1 B evict_last, CSR/C evict_first; 2 = 1 but
                                    # cold B rows (hot-column map) evict_normal
    hub_threshold: int = 0          # 0 auto, <0 off
    l2_persist: int = 0             # 1 L2 access-policy window marking B persisting; 2 set-aside only
    l2_hot_mb: int = 0              # hot-column map budget in MB: 0 auto (off), <0 off
    tuned_cf: int = 0               # tuned warp kernel merge factor (1/2/4), 0 auto
    col_slices: int = 0             # slice-major column traversal: 0 auto, 1 off, S slices
    rows_per_warp: int = 0          # rows sharing a warp (float4 lanes, N <= 256): 0 auto
    cluster_hot: int = 0            # N = 128 plans: hot B rows in cluster DSMEM (cluster size), 0 off
    h2d_pack: int = 0               # host entry: 16-bit gap codes for col_ind upload; 0 auto, 1 on, -1 off
    hot_rows_mb: int = 0            # relocated hot B rows (plan-owned copy), MB; <=0 off (experimental)
    overlap_prev: bool = False      # single-kernel plans: programmatic dependent launch onto the
                                    # previous kernel (A prologue before the wait; gespmm.h contract)


def _options(variant: KernelVariant, ex: ExecOptions, validate: bool = True) -> _lib.Options:
    return default_options(variant=int(variant.kind), cf=variant.cf if variant.cf else 2,
                           exact=int(ex.exact),
                           arg_kind=_lib.ARG_COLUMN if ex.arg_kind == "column" else _lib.ARG_EDGE,
                           validate=int(validate), fault_skip_tail=int(ex.fault == FaultMode.SkipTail),
                           l2_hints=int(ex.l2_hints), hub_threshold=ex.hub_threshold,
                           l2_persist=int(ex.l2_persist), l2_hot_mb=int(ex.l2_hot_mb),
                           tuned_cf=int(ex.tuned_cf), col_slices=int(ex.col_slices),
                           rows_per_warp=int(ex.rows_per_warp), cluster_hot=int(ex.cluster_hot),
                           h2d_pack=int(ex.h2d_pack), hot_rows_mb=int(ex.hot_rows_mb),
                           overlap_prev=int(ex.overlap_prev))


# ---------------------------------------------------------------------------
# the hot path: native_spmm-shaped host call
# ---------------------------------------------------------------------------

def _length_checks(a: CsrMatrix):
    """The two validate() checks a C struct cannot express (csr.hpp:116-123)."""
    pre = "spmm: matrix is not canonical CSR: "
    if len(a.row_ptr) != a.n_rows + 1:
        raise Error(pre + f"row_ptr length is {len(a.row_ptr)}, expected n_rows+1 = "
                    f"{a.n_rows + 1}", _lib.ENONCANON)
    if len(a.col_ind) != len(a.vals):
        raise Error(pre + f"col_ind length {len(a.col_ind)} != vals length {len(a.vals)}",
                    _lib.ENONCANON)


def native_spmm_arg(a: CsrMatrix, b: DenseMatrix, variant: KernelVariant, op: ReduceOp,
                    workers: int = 0, exec: ExecOptions = ExecOptions(),
                    want_arg: bool = False) -> Tuple[DenseMatrix, Optional[np.ndarray]]:
    """native_spmm plus argmax/argmin indices (int32, -1 = none) for max/min."""
    del workers
    check_dense_valid(b)
    if a.n_cols != b.n_rows:
        raise Error(f"spmm: dimension mismatch: A is {a.n_rows}x{a.n_cols} but B has "
                    f"{b.n_rows} rows", _lib.EDIM)
    _length_checks(a)
    csr, keep = a._c()
    bd = np.ascontiguousarray(b.data, np.float32)
    n = b.n_cols
    c = np.empty((a.n_rows, n), np.float32)
    arg = np.empty((a.n_rows, n), np.int32) if want_arg else None
    o = _options(variant, exec)
    st = lib().gespmm_spmm_host(C.byref(csr), bd.ctypes.data if bd.size else None, b.n_rows, n,
                                op.code, c.ctypes.data if c.size else None,
                                arg.ctypes.data if arg is not None and arg.size else None,
                                C.byref(o))
    del keep
    _check(st)
    return DenseMatrix(a.n_rows, n, c), arg


def native_spmm(a: CsrMatrix, b: DenseMatrix, variant: KernelVariant, op: ReduceOp,
                workers: int = 0, exec: ExecOptions = ExecOptions()) -> DenseMatrix:
    """native.hpp:101-143 on the B200: validate, H2D, kernel, D2H."""
    return native_spmm_arg(a, b, variant, op, workers, exec)[0]


@dataclasses.dataclass
class ThroughputReport:
    """native.hpp:147-154."""
    elapsed_s: float = 0.0
    elapsed_mean_s: float = 0.0
    repeats: int = 0
    flops: int = 0
    gflops: float = 0.0
    output_checksum: int = 0


def bench(a: CsrMatrix, b: DenseMatrix, variant: KernelVariant, op: ReduceOp, workers: int = 0,
          repeats: int = 9) -> ThroughputReport:
    """native.hpp:156-180: median wall time of native_spmm, theoretical 2*nnz*N flops,
    checksum outside the timed window."""
    if repeats < 1:
        raise Error("bench: repeats must be >= 1")
    rep = ThroughputReport(repeats=repeats, flops=2 * a.nnz() * b.n_cols)
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        c = native_spmm(a, b, variant, op, workers)
        times.append(time.perf_counter() - t0)
        rep.output_checksum = checksum(c)
    times.sort()
    rep.elapsed_s = times[(len(times) - 1) // 2]
    rep.elapsed_mean_s = sum(times) / len(times)
    rep.gflops = rep.flops / rep.elapsed_s / 1e9 if rep.elapsed_s > 0 else 0.0
    return rep


# ---------------------------------------------------------------------------
# inputs and checksum (host C++ in the library)
# ---------------------------------------------------------------------------

def checksum(m: DenseMatrix) -> int:
    d = np.ascontiguousarray(m.data, np.float32)
    return int(lib().gespmm_checksum(d.ctypes.data, m.n_rows, m.n_cols))


def make_random_dense(rows: int, cols: int, seed: int) -> DenseMatrix:
    out = np.empty((rows, cols), np.float32)
    if out.size:
        lib().gespmm_make_random_dense(rows, cols, seed, out.ctypes.data)
    return DenseMatrix(rows, cols, out)


def randomize_values(m: CsrMatrix, seed: int) -> None:
    v = np.ascontiguousarray(m.vals, np.float32)
    if v.size:
        lib().gespmm_randomize_values(v.ctypes.data, v.size, seed)
    m.vals = v


@dataclasses.dataclass(frozen=True)
class GraphGenSpec:
    n_rows: int = 0
    nnz_target: int = 0
    seed: int = 0
    self_loops: bool = False


def gen_uniform_random(spec: GraphGenSpec) -> CsrMatrix:
    rp = np.zeros(spec.n_rows + 1, np.uint32)
    ci = np.empty(max(spec.nnz_target, 1), np.uint32)
    v = np.empty(max(spec.nnz_target, 1), np.float32)
    _check(lib().gespmm_gen_uniform(spec.n_rows, spec.nnz_target, spec.seed, int(spec.self_loops),
                                    rp.ctypes.data, ci.ctypes.data, v.ctypes.data))
    return CsrMatrix(spec.n_rows, spec.n_rows, rp, ci[:spec.nnz_target], v[:spec.nnz_target])


def gen_powerlaw(n_rows: int, nnz_target: int, max_degree: int, exponent: float = 1.0,
                 seed: int = 1, threads: int = 0) -> CsrMatrix:
    """Deterministic Chung-Lu-style power-law square graph (new; see gespmm.h)."""
    rp = np.zeros(n_rows + 1, np.uint32)
    L = lib()
    _check(L.gespmm_gen_powerlaw(n_rows, nnz_target, max_degree, exponent, seed, threads,
                                 rp.ctypes.data, None, None))
    nnz = int(rp[-1])
    ci = np.empty(max(nnz, 1), np.uint32)
    v = np.empty(max(nnz, 1), np.float32)
    _check(L.gespmm_gen_powerlaw(n_rows, nnz_target, max_degree, exponent, seed, threads,
                                 rp.ctypes.data, ci.ctypes.data, v.ctypes.data))
    return CsrMatrix(n_rows, n_rows, rp, ci[:nnz], v[:nnz])


# ---------------------------------------------------------------------------
# CSR1 binary cache (io.hpp:15-16, 50-115)
# ---------------------------------------------------------------------------

def _path_bytes(path) -> bytes:
    import os
    return os.fsencode(path)


def save_csr_cache(path, m: CsrMatrix) -> None:
    """save_csr_cache / write_csr_cache (io.hpp:50-63, 92-96)."""
    s, _keep = m._c()
    _check(lib().gespmm_csr1_write(_path_bytes(path), C.byref(s)))


def _csr1_header(path) -> Tuple[int, int, int]:
    r, c, z = C.c_uint32(), C.c_uint32(), C.c_uint64()
    _check(lib().gespmm_csr1_header(_path_bytes(path), C.byref(r), C.byref(c), C.byref(z)))
    return r.value, c.value, z.value


def read_csr_cache(path) -> CsrMatrix:
    """read_csr_cache (io.hpp:65-90): no canonical check (as the reference)."""
    rows, cols, nnz = _csr1_header(path)
    rp = np.empty(rows + 1, np.uint32)
    ci = np.empty(nnz, np.uint32)
    v = np.empty(nnz, np.float32)
    _check(lib().gespmm_csr1_read_host(_path_bytes(path), rp.ctypes.data, ci.ctypes.data,
                                       v.ctypes.data))
    return CsrMatrix(rows, cols, rp, ci, v)


def load_matrix(path) -> CsrMatrix:
    """load_matrix (io.hpp:100-115): .mtx parses Matrix Market and canonicalises
    with duplicate summation, .csr reads the binary cache; both then get the
    canonical check with the reference's "load_matrix: matrix is not canonical
    CSR: ..." text."""
    import os
    ext = os.path.splitext(os.fspath(path))[1]
    if ext not in (".mtx", ".csr"):
        if not os.path.exists(path):
            raise Error(f"cannot open '{os.fspath(path)}'")
        raise Error(f"unknown matrix extension '{ext}' (expected .mtx or .csr)")
    if ext == ".mtx":
        try:
            with open(path, "rb") as f:
                text = f.read()
        except OSError:
            raise Error(f"cannot open '{os.fspath(path)}'") from None
        rows, cols, triples = parse_matrix_market(text)
        m = from_coo(rows, cols, triples, "sum")
    else:
        m = read_csr_cache(path)
    require_canonical(m, "load_matrix")
    return m


def _host_validate(m: CsrMatrix, who: str) -> None:
    """Canonical check of a host CSR on the device (validate, csr.hpp:112-153)."""
    import torch
    if not torch.cuda.is_available():
        raise Error(f"{who}: no CUDA device for the canonical check", _lib.ECUDA)
    d = DeviceCsr.from_host(m, "cuda")
    _check(lib().gespmm_validate_device_as(C.byref(d.c_struct()), _stream_ptr(None),
                                           who.encode()))


# ---------------------------------------------------------------------------
# device-resident API (torch tensors for memory/streams only)
# ---------------------------------------------------------------------------

class DeviceCsr:
    """A CSR whose arrays live in HBM (torch uint32/int32 + float32 tensors)."""

    def __init__(self, n_rows, n_cols, row_ptr, col_ind, vals):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr, self.col_ind, self.vals = row_ptr, col_ind, vals

    @classmethod
    def from_host(cls, a: CsrMatrix, device="cuda") -> "DeviceCsr":
        import torch
        rp = torch.from_numpy(np.ascontiguousarray(a.row_ptr, np.uint32).view(np.int32)).to(device)
        ci = torch.from_numpy(np.ascontiguousarray(a.col_ind, np.uint32).view(np.int32)).to(device)
        v = torch.from_numpy(np.ascontiguousarray(a.vals, np.float32)).to(device)
        return cls(a.n_rows, a.n_cols, rp, ci, v)

    @classmethod
    def load(cls, path, device="cuda", validate: bool = True, stream=None) -> "DeviceCsr":
        """Stream a CSR1 cache file straight into HBM (gespmm_csr1_load_device:
        pinned double-buffered reads overlapped with H2D), then the device
        canonical check with load_matrix's wording (io.hpp:100-115)."""
        import torch
        rows, cols, nnz = _csr1_header(path)
        rp = torch.empty(rows + 1, dtype=torch.int32, device=device)
        ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=device)
        v = torch.empty(max(nnz, 1), dtype=torch.float32, device=device)
        with torch.cuda.device(rp.device):
            _check(lib().gespmm_csr1_load_device(_path_bytes(path), rp.data_ptr(), ci.data_ptr(),
                                                 v.data_ptr(), int(validate), _stream_ptr(stream)))
        return cls(rows, cols, rp, ci[:nnz], v[:nnz])

    @classmethod
    def from_coo(cls, n_rows: int, n_cols: int, rows, cols, vals, policy: str = "sum",
                 stream=None) -> "DeviceCsr":
        """from_coo (csr.hpp:58-93) on device triples (torch int32/uint32 and
        float32 tensors on one CUDA device) through gespmm_from_coo_device:
        bit-identical to the host from_coo, errors worded like the reference."""
        import torch
        if policy not in ("sum", "last"):
            raise Error(f"from_coo: unknown dedup policy '{policy}' (sum, last)")
        n = int(rows.numel())
        if int(cols.numel()) != n or int(vals.numel()) != n:
            raise Error("from_coo: rows, cols and vals must have the same length")
        for t, dt, what in ((rows, (torch.int32,), "rows"), (cols, (torch.int32,), "cols"),
                            (vals, (torch.float32,), "vals")):
            if not t.is_cuda or t.dtype not in dt or not t.is_contiguous():
                raise Error(f"from_coo: {what} must be a contiguous CUDA {dt[0]} tensor")
        dev = rows.device
        rp = torch.empty(n_rows + 1, dtype=torch.int32, device=dev)
        ci = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        v = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        nnz = C.c_uint64()
        with torch.cuda.device(dev):
            _check(lib().gespmm_from_coo_device(
                n_rows, n_cols, n, rows.data_ptr() if n else None, cols.data_ptr() if n else None,
                vals.data_ptr() if n else None, 0 if policy == "sum" else 1, rp.data_ptr(),
                ci.data_ptr(), v.data_ptr(), C.byref(nnz), _stream_ptr(stream)))
        z = int(nnz.value)
        return cls(n_rows, n_cols, rp, ci[:z], v[:z])

    def to_coo(self, stream=None):
        """(rows, cols, vals) device tensors in row-major order (csr.hpp:95-104)."""
        import torch
        dev = self.row_ptr.device
        n = self.nnz()
        r = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        c = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        v = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        csr = self.c_struct()
        with torch.cuda.device(dev):
            _check(lib().gespmm_to_coo_device(C.byref(csr), r.data_ptr(), c.data_ptr(),
                                              v.data_ptr(), _stream_ptr(stream)))
        return r[:n], c[:n], v[:n]

    def nnz(self) -> int:
        return int(self.col_ind.numel())

    def transpose(self, stream=None) -> "DeviceCsr":
        """A^T as a canonical device CSR (gespmm_csr_transpose_device)."""
        import torch
        dev = self.row_ptr.device
        rp = torch.empty(self.n_cols + 1, dtype=torch.int32, device=dev)
        ci = torch.empty(max(self.nnz(), 1), dtype=torch.int32, device=dev)
        v = torch.empty(max(self.nnz(), 1), dtype=torch.float32, device=dev)
        csr = self.c_struct()
        _check(lib().gespmm_csr_transpose_device(C.byref(csr), rp.data_ptr(), ci.data_ptr(),
                                                 v.data_ptr(), _stream_ptr(stream)))
        return DeviceCsr(self.n_cols, self.n_rows, rp, ci[: self.nnz()], v[: self.nnz()])

    def to_host(self) -> CsrMatrix:
        return CsrMatrix(self.n_rows, self.n_cols,
                         self.row_ptr.cpu().numpy().view(np.uint32).copy(),
                         self.col_ind.cpu().numpy().view(np.uint32).copy(),
                         self.vals.cpu().numpy().copy())

    def c_struct(self) -> Csr:
        return Csr(self.n_rows, self.n_cols, self.nnz(), self.row_ptr.data_ptr(),
                   self.col_ind.data_ptr() if self.nnz() else None,
                   self.vals.data_ptr() if self.nnz() else None)


def _require_dense(t, rows: int, cols: int, dtype, device, what: str):
    """Raw device pointers go to the kernels: refuse anything that is not a
    contiguous 2-D tensor of exactly the plan's shape, dtype and device."""
    import torch
    ok = (isinstance(t, torch.Tensor) and t.dim() == 2 and t.dtype == dtype and t.is_cuda
          and t.is_contiguous() and tuple(t.shape) == (rows, cols)
          and (device is None or t.device == device))
    if not ok:
        got = (f"{tuple(t.shape)} {t.dtype} on {t.device}"
               f"{'' if t.is_contiguous() else ' (non-contiguous)'}"
               if isinstance(t, torch.Tensor) else type(t).__name__)
        raise Error(f"{what}: expected a contiguous {rows}x{cols} {dtype} CUDA tensor"
                    f"{'' if device is None else f' on {device}'}, got {got}", _lib.EDIM)


def _stream_ptr(stream=None) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def release_workspace():
    """gespmm_release_workspace: free the library's grow-only scratch (host
    entry staging, COO builder temporaries) on the current device."""
    lib().gespmm_release_workspace()


def spmm(a: DeviceCsr, b, op: ReduceOp | str = "sum", want_arg: bool = False,
         variant: KernelVariant = KernelVariant.tuned(), exec: ExecOptions = ExecOptions(),
         validate: bool = True, out=None, stream=None):
    """C = A (x) B on the device; returns (C, arg or None) as torch tensors.
    ``validate`` (default on, like the reference's native_spmm) runs the
    canonical-CSR check on the device first."""
    import torch
    if isinstance(op, str):
        op = reduce_op_by_name(op)
    if b.dim() != 2 or b.dtype != torch.float32 or not b.is_cuda:
        raise Error("spmm: B must be a 2-D float32 CUDA tensor")
    b = b.contiguous()
    if b.shape[0] != a.n_cols:
        raise Error(f"spmm: dimension mismatch: A is {a.n_rows}x{a.n_cols} but B has "
                    f"{b.shape[0]} rows", _lib.EDIM)
    n = b.shape[1]
    if a.row_ptr.device != b.device:
        raise Error(f"spmm: A is on {a.row_ptr.device} but B is on {b.device}", _lib.EDIM)
    if out is not None:
        _require_dense(out, a.n_rows, n, torch.float32, b.device, "spmm: out")
    c = out if out is not None else torch.empty((a.n_rows, n), dtype=torch.float32, device=b.device)
    arg = torch.empty((a.n_rows, n), dtype=torch.int32, device=b.device) if want_arg else None
    csr = a.c_struct()
    o = _options(variant, exec, validate)
    _check(lib().gespmm_spmm_device(C.byref(csr), b.data_ptr(), n, op.code, c.data_ptr(),
                                    arg.data_ptr() if arg is not None else None, C.byref(o),
                                    _stream_ptr(stream)))
    return c, arg


class Plan:
    """gespmm_plan_*: inspect A once (degree distribution -> kernel shapes and
    row schedule), execute many times.  ``launches`` kernels per execute."""

    def __init__(self, a: DeviceCsr, n: int, op: ReduceOp | str = "sum",
                 variant: KernelVariant = KernelVariant.tuned(),
                 exec: ExecOptions = ExecOptions(), stream=None):
        if isinstance(op, str):
            op = reduce_op_by_name(op)
        self.a, self.n, self.op = a, int(n), op
        self._csr = a.c_struct()
        o = _options(variant, exec, validate=False)
        h = C.c_void_p()
        _check(lib().gespmm_plan_create(C.byref(self._csr), self.n, op.code, C.byref(o),
                                        _stream_ptr(stream), C.byref(h)))
        self._h = h

    @property
    def description(self) -> str:
        return lib().gespmm_plan_describe(self._h).decode()

    @property
    def launches(self) -> int:
        return int(lib().gespmm_plan_launches(self._h))

    def _check_operands(self, b, c=None, arg=None):
        import torch
        dev = self.a.row_ptr.device
        _require_dense(b, self.a.n_cols, self.n, torch.float32, dev, "Plan: B")
        if c is not None:
            _require_dense(c, self.a.n_rows, self.n, torch.float32, dev, "Plan: C")
        if arg is not None:
            _require_dense(arg, self.a.n_rows, self.n, torch.int32, dev, "Plan: arg")

    def execute(self, b, c, arg=None, stream=None):
        self._check_operands(b, c, arg)
        _check(lib().gespmm_plan_execute(self._h, b.data_ptr(), c.data_ptr(),
                                         arg.data_ptr() if arg is not None else None,
                                         _stream_ptr(stream)))
        return c

    def execute_gather(self, b, c_dsts, arg_dsts=None, c_multicast=None, arg_multicast=None,
                       stream=None):
        """gespmm_plan_execute_gather: the plan's SpMM with its output rows also
        stored into replicas (fused all-gather epilogue).  ``c_dsts`` are raw
        device addresses (ints) of where this shard's row 0 lands, local first;
        ``arg_dsts`` likewise for max/min arg (or None)."""
        self._check_operands(b)
        k = len(c_dsts)
        cd = (C.c_void_p * k)(*[int(x) for x in c_dsts])
        ad = None
        if arg_dsts is not None:
            ad = (C.c_void_p * k)(*[int(x) if x else None for x in arg_dsts])
        _check(lib().gespmm_plan_execute_gather(self._h, b.data_ptr(), cd, ad, k,
                                                int(c_multicast) if c_multicast else None,
                                                int(arg_multicast) if arg_multicast else None,
                                                _stream_ptr(stream)))

    def close(self):
        if getattr(self, "_h", None):
            lib().gespmm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_info() -> dict:
    sm, l2, pl2, ma, mi = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32()
    _check(lib().gespmm_device_info(C.byref(sm), C.byref(l2), C.byref(pl2), C.byref(ma),
                                    C.byref(mi)))
    return {"sm_count": sm.value, "l2_bytes": l2.value, "persisting_l2_max": pl2.value,
            "cc": f"{ma.value}.{mi.value}"}
