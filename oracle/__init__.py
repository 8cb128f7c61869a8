"""TEST INFRASTRUCTURE ONLY — CPU oracle for the GE-SpMM hot path.

Two checkers live here, both loaded with ctypes:

* ``restatement`` — ``liboracle.so`` built from ``oracle/spmm_oracle.c``: the
  reference's ordered fold restated in plain C (sum / mean / max / min and
  argmax/argmin), plus the canonical-CSR validator and the FNV-1a checksum.
* ``reference`` — ``_ref/libspmmref.so``: the UNMODIFIED reference headers
  (``/root/reference/proj/include/spmm``) compiled in place by
  ``oracle/Makefile`` behind ``oracle/ref_shim.cpp``.  Present in the dev
  container and wherever the prebuilt .so travelled; absent otherwise.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product (``paper_2007_03179_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspmmref.so")

OPS = {"sum": 0, "mean": 1, "max": 2, "min": 3}
ARG_EDGE, ARG_COLUMN = 0, 1
KIND = {"naive": 0, "crc": 1, "crc-cwm": 2}

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")

_oracle = None
_ref = None


def build() -> None:
    """Compile the restatement (and the reference shim when /root/reference exists)."""
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


def _load_oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        lib.oracle_spmm.restype = C.c_int
        lib.oracle_spmm.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p, _f32p, _f32p,
                                    C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int,
                                    _f32p, C.c_void_p]
        lib.oracle_checksum.restype = C.c_uint64
        lib.oracle_checksum.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p]
        lib.oracle_gen_powerlaw.restype = C.c_int
        lib.oracle_gen_powerlaw.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_double,
                                            C.c_uint64, C.c_int, _u32p, C.c_void_p, C.c_void_p]
        lib.oracle_make_random_dense.restype = None
        lib.oracle_make_random_dense.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p]
        lib.oracle_randomize_values.restype = None
        lib.oracle_randomize_values.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        lib.oracle_validate.restype = C.c_int
        lib.oracle_validate.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_uint64, _u32p,
                                        C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint32]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _load_ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"reference shim not built: {REF_SO}")
        lib = C.CDLL(REF_SO)
        cp, cu, cull, cd = C.c_char_p, C.c_uint, C.c_ulonglong, C.c_double
        lib.ref_native_spmm.restype = C.c_int
        lib.ref_native_spmm.argtypes = [cu, cu, cull, _u32p, _u32p, _f32p, _f32p, cu, cp,
                                        C.c_int, cu, cu, C.c_int, _f32p, cp, cu]
        lib.ref_native_spmm_shape.restype = C.c_int
        lib.ref_native_spmm_shape.argtypes = [cu, cu, cull, _u32p, cu, _u32p, cull, _f32p,
                                              cull, _f32p, cu, cu, cp, cp, cu]
        lib.ref_bench.restype = C.c_int
        lib.ref_bench.argtypes = [cu, cu, cull, _u32p, _u32p, _f32p, _f32p, cu, cp, C.c_int,
                                  cu, cu, cu, C.POINTER(cd), C.POINTER(cd), C.POINTER(cd),
                                  C.POINTER(cull), cp, cu]
        lib.ref_dense_reference.restype = C.c_int
        lib.ref_dense_reference.argtypes = [cu, cu, cull, _u32p, _u32p, _f32p, _f32p, cu, cp,
                                            _f32p, cp, cu]
        lib.ref_gen_uniform.restype = C.c_int
        lib.ref_gen_uniform.argtypes = [cu, cull, cull, C.c_int, _u32p, _u32p, _f32p, cp, cu]
        lib.ref_randomize_values.restype = None
        lib.ref_randomize_values.argtypes = [_f32p, cull, cull]
        lib.ref_make_random_dense.restype = None
        lib.ref_make_random_dense.argtypes = [cu, cu, cull, _f32p]
        lib.ref_checksum.restype = cull
        lib.ref_checksum.argtypes = [cu, cu, _f32p]
        lib.ref_validate.restype = C.c_int
        lib.ref_validate.argtypes = [cu, cu, _u32p, cu, _u32p, cull, _f32p, cull, cp, cu]
        lib.ref_select_variant.restype = None
        lib.ref_select_variant.argtypes = [cu, C.POINTER(C.c_int), C.POINTER(cu)]
        lib.ref_from_coo.restype = C.c_longlong
        lib.ref_from_coo.argtypes = [cu, cu, cull, _u32p, _u32p, _f32p, _u32p, _u32p, _f32p,
                                     cp, cu, C.c_int]
        lib.ref_sim_metrics.restype = C.c_int
        lib.ref_sim_metrics.argtypes = [cu, cu, cull, _u32p, _u32p, _f32p, _f32p, cu, cp,
                                        C.c_int, cu, C.POINTER(cull), cp, cu]
        lib.ref_save_csr_cache.restype = C.c_int
        lib.ref_save_csr_cache.argtypes = [cp, cu, cu, cull, _u32p, _u32p, _f32p, cp, cu]
        lib.ref_load_matrix.restype = C.c_int
        lib.ref_load_matrix.argtypes = [cp, C.POINTER(cu), C.POINTER(cu), C.POINTER(cull),
                                        C.c_void_p, C.c_void_p, C.c_void_p, cp, cu]
        lib.ref_session_new.restype = C.c_void_p
        lib.ref_session_new.argtypes = [cu, cu, cull, _u32p, _u32p, _f32p, _f32p, cu, cp, cu]
        lib.ref_session_bench.restype = C.c_int
        lib.ref_session_bench.argtypes = [C.c_void_p, cp, C.c_int, cu, cu, cu, C.POINTER(cd),
                                          C.POINTER(cd), C.POINTER(cd), C.POINTER(cull), cp, cu]
        lib.ref_session_free.restype = None
        lib.ref_session_free.argtypes = [C.c_void_p]
        lib.ref_hardware_concurrency.restype = cu
        lib.ref_hardware_concurrency.argtypes = []
        _ref = lib
    return _ref


class RefError(RuntimeError):
    """An exception raised by the reference (spmm::Error text preserved)."""


# --------------------------------------------------------------------------
# restatement
# --------------------------------------------------------------------------

def spmm(m, k, row_ptr, col_ind, vals, b, op="sum", want_arg=False, arg_kind=ARG_EDGE,
         skip_tail=False, threads=None):
    """Ordered-fold restatement; returns C (m x n float32) and arg (int32) or None."""
    lib = _load_oracle()
    b = np.ascontiguousarray(b, dtype=np.float32)
    n = b.shape[1] if b.ndim == 2 else 0
    c = np.empty((m, n), dtype=np.float32)
    arg = np.empty((m, n), dtype=np.int32) if want_arg else None
    if threads is None:
        threads = os.cpu_count() or 1
    rc = lib.oracle_spmm(m, k, np.ascontiguousarray(row_ptr, np.uint32),
                         np.ascontiguousarray(col_ind, np.uint32),
                         np.ascontiguousarray(vals, np.float32), b.reshape(-1) if b.size else
                         np.zeros(1, np.float32), n, OPS[op], arg_kind, int(skip_tail),
                         int(threads), c.reshape(-1) if c.size else np.zeros(1, np.float32),
                         arg.ctypes.data if arg is not None else None)
    if rc != 0:
        raise ValueError("oracle_spmm: bad arguments")
    return c, arg


def gen_powerlaw(rows, nnz_target, max_degree, exponent=1.0, seed=1, threads=None):
    """Restatement of the benchmark's power-law generator (powerlaw_oracle.c);
    returns (row_ptr, col_ind, vals) — bit-identical to the product's
    gen_powerlaw, built without loading the product library."""
    lib = _load_oracle()
    threads = threads or os.cpu_count() or 1
    rp = np.zeros(rows + 1, np.uint32)
    rc = lib.oracle_gen_powerlaw(rows, nnz_target, max_degree, exponent, seed, threads, rp,
                                 None, None)
    if rc:
        raise ValueError(f"oracle_gen_powerlaw: rc {rc}")
    nnz = int(rp[-1])
    ci = np.empty(max(nnz, 1), np.uint32)
    v = np.empty(max(nnz, 1), np.float32)
    rc = lib.oracle_gen_powerlaw(rows, nnz_target, max_degree, exponent, seed, threads, rp,
                                 ci.ctypes.data, v.ctypes.data)
    if rc:
        raise ValueError(f"oracle_gen_powerlaw: rc {rc}")
    return rp, ci[:nnz], v[:nnz]


def make_random_dense(rows, cols, seed):
    """dense.hpp:51-59 restated (MT19937-64 in C)."""
    out = np.empty((rows, cols), np.float32)
    if out.size:
        _load_oracle().oracle_make_random_dense(rows, cols, seed, out.ctypes.data)
    return out


def randomize_values(vals, seed):
    """generate.hpp:73-80 restated; fills ``vals`` (float32, contiguous) in place."""
    assert vals.dtype == np.float32 and vals.flags.c_contiguous
    if vals.size:
        _load_oracle().oracle_randomize_values(vals.ctypes.data, vals.size, seed)
    return vals


def checksum(c: np.ndarray) -> int:
    c = np.ascontiguousarray(c, dtype=np.float32)
    rows, cols = (c.shape if c.ndim == 2 else (c.shape[0], 1))
    return int(_load_oracle().oracle_checksum(rows, cols, c.ctypes.data))


def validate(m, k, row_ptr, col_ind, vals):
    """(violation_count, first_message) per the reference's csr.hpp validate()."""
    buf = C.create_string_buffer(512)
    rp = np.ascontiguousarray(row_ptr, np.uint32)
    ci = np.ascontiguousarray(col_ind, np.uint32)
    if rp.size == 0:
        rp = np.zeros(1, np.uint32)
        rp_len = 0
    else:
        rp_len = rp.size
    n = _load_oracle().oracle_validate(m, k, rp, rp_len, ci if ci.size else np.zeros(1, np.uint32),
                                       ci.size, len(vals), buf, 512)
    return n, buf.value.decode()


# --------------------------------------------------------------------------
# reference (unmodified, via the shim)
# --------------------------------------------------------------------------

def _err():
    return C.create_string_buffer(1024)


def _nz(a, dt):
    a = np.ascontiguousarray(a, dt)
    return a if a.size else np.zeros(1, dt)


def ref_native_spmm(m, k, row_ptr, col_ind, vals, b, op="sum", variant="crc", cf=2,
                    workers=1, skip_tail=False):
    lib = _load_ref()
    b = np.ascontiguousarray(b, np.float32)
    n = b.shape[1]
    c = np.empty((m, n), np.float32)
    e = _err()
    rc = lib.ref_native_spmm(m, k, len(col_ind), _nz(row_ptr, np.uint32), _nz(col_ind, np.uint32),
                             _nz(vals, np.float32), _nz(b.reshape(-1), np.float32), n,
                             op.encode(), KIND[variant], cf, workers, int(skip_tail),
                             _nz(c.reshape(-1), np.float32) if c.size == 0 else c.reshape(-1),
                             e, 1024)
    if rc:
        raise RefError(e.value.decode())
    return c


def ref_bench(m, k, row_ptr, col_ind, vals, b, op="sum", variant="crc-cwm", cf=2, workers=0,
              repeats=3):
    lib = _load_ref()
    b = np.ascontiguousarray(b, np.float32)
    med, mean, gf = C.c_double(), C.c_double(), C.c_double()
    cs = C.c_ulonglong()
    e = _err()
    rc = lib.ref_bench(m, k, len(col_ind), _nz(row_ptr, np.uint32), _nz(col_ind, np.uint32),
                       _nz(vals, np.float32), _nz(b.reshape(-1), np.float32), b.shape[1],
                       op.encode(), KIND[variant], cf, workers, repeats, C.byref(med),
                       C.byref(mean), C.byref(gf), C.byref(cs), e, 1024)
    if rc:
        raise RefError(e.value.decode())
    return {"median_s": med.value, "mean_s": mean.value, "gflops": gf.value,
            "checksum": cs.value}


class RefSession:
    """The reference's CsrMatrix + DenseMatrix built once; ``bench()`` runs
    spmm::bench (native.hpp:156-180) on them, so only the reference's own
    timing window is measured."""

    def __init__(self, m, k, row_ptr, col_ind, vals, b):
        lib = _load_ref()
        b = np.ascontiguousarray(b, np.float32)
        self.n = b.shape[1]
        e = _err()
        self._h = lib.ref_session_new(m, k, len(col_ind), _nz(row_ptr, np.uint32),
                                      _nz(col_ind, np.uint32), _nz(vals, np.float32),
                                      _nz(b.reshape(-1), np.float32), self.n, e, 1024)
        if not self._h:
            raise RefError(e.value.decode())

    def bench(self, op="sum", variant="crc-cwm", cf=2, workers=0, repeats=1):
        med, mean, gf = C.c_double(), C.c_double(), C.c_double()
        cs = C.c_ulonglong()
        e = _err()
        if _load_ref().ref_session_bench(self._h, op.encode(), KIND[variant], cf, workers,
                                         repeats, C.byref(med), C.byref(mean), C.byref(gf),
                                         C.byref(cs), e, 1024):
            raise RefError(e.value.decode())
        return {"median_s": med.value, "mean_s": mean.value, "gflops": gf.value,
                "checksum": cs.value}

    def close(self):
        if getattr(self, "_h", None):
            _load_ref().ref_session_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_dense_reference(m, k, row_ptr, col_ind, vals, b, op="sum"):
    lib = _load_ref()
    b = np.ascontiguousarray(b, np.float32)
    c = np.empty((m, b.shape[1]), np.float32)
    e = _err()
    rc = lib.ref_dense_reference(m, k, len(col_ind), _nz(row_ptr, np.uint32),
                                 _nz(col_ind, np.uint32), _nz(vals, np.float32),
                                 _nz(b.reshape(-1), np.float32), b.shape[1], op.encode(),
                                 c.reshape(-1), e, 1024)
    if rc:
        raise RefError(e.value.decode())
    return c


def ref_gen_uniform(rows, nnz, seed, self_loops=False):
    lib = _load_ref()
    rp = np.zeros(rows + 1, np.uint32)
    ci = np.zeros(max(nnz, 1), np.uint32)
    v = np.zeros(max(nnz, 1), np.float32)
    e = _err()
    if lib.ref_gen_uniform(rows, nnz, seed, int(self_loops), rp if rows + 1 else _nz(rp, np.uint32),
                           ci, v, e, 1024):
        raise RefError(e.value.decode())
    return rp, ci[:nnz].copy(), v[:nnz].copy()


def ref_randomize_values(vals, seed):
    v = np.ascontiguousarray(vals, np.float32).copy()
    if v.size:
        _load_ref().ref_randomize_values(v, v.size, seed)
    return v


def ref_make_random_dense(rows, cols, seed):
    out = np.zeros((rows, cols), np.float32)
    if out.size:
        _load_ref().ref_make_random_dense(rows, cols, seed, out.reshape(-1))
    return out


def ref_checksum(c):
    c = np.ascontiguousarray(c, np.float32)
    return int(_load_ref().ref_checksum(c.shape[0], c.shape[1], _nz(c.reshape(-1), np.float32)))


def ref_validate(m, k, row_ptr, col_ind, vals):
    buf = C.create_string_buffer(512)
    n = _load_ref().ref_validate(m, k, _nz(row_ptr, np.uint32), len(row_ptr),
                                 _nz(col_ind, np.uint32), len(col_ind), _nz(vals, np.float32),
                                 len(vals), buf, 512)
    return n, buf.value.decode()


def ref_native_spmm_error(m, k, row_ptr, col_ind, vals, b, b_rows, n, op="sum"):
    """Run native_spmm on possibly-invalid inputs; return the error text or None."""
    e = _err()
    rc = _load_ref().ref_native_spmm_shape(
        m, k, len(col_ind), _nz(row_ptr, np.uint32), len(row_ptr), _nz(col_ind, np.uint32),
        len(col_ind), _nz(vals, np.float32), len(vals), _nz(np.asarray(b).reshape(-1), np.float32),
        b_rows, n, op.encode(), e, 1024)
    return e.value.decode() if rc else None


def ref_select_variant(n):
    kind, cf = C.c_int(), C.c_uint()
    _load_ref().ref_select_variant(n, C.byref(kind), C.byref(cf))
    return {0: "naive", 1: "crc", 2: "crc-cwm"}[kind.value], cf.value


def ref_from_coo(rows, cols, r, c, v, policy="sum"):
    cnt = len(r)
    rp = np.zeros(rows + 1, np.uint32)
    ci = np.zeros(max(cnt, 1), np.uint32)
    vv = np.zeros(max(cnt, 1), np.float32)
    e = _err()
    nnz = _load_ref().ref_from_coo(rows, cols, cnt, _nz(r, np.uint32), _nz(c, np.uint32),
                                   _nz(v, np.float32), rp, ci, vv, e, 1024,
                                   0 if policy == "sum" else 1)
    if nnz < 0:
        raise RefError(e.value.decode())
    return rp, ci[:nnz].copy(), vv[:nnz].copy()


def ref_hardware_concurrency():
    return int(_load_ref().ref_hardware_concurrency())


def ref_save_csr_cache(path, m, k, row_ptr, col_ind, vals):
    e = _err()
    if _load_ref().ref_save_csr_cache(os.fsencode(path), m, k, len(col_ind),
                                      _nz(row_ptr, np.uint32), _nz(col_ind, np.uint32),
                                      _nz(vals, np.float32), e, 1024):
        raise RefError(e.value.decode())


def ref_load_matrix(path):
    """The reference's load_matrix (read + require_canonical); (m, k, rp, ci, v)."""
    lib = _load_ref()
    m, k, z = C.c_uint(), C.c_uint(), C.c_ulonglong()
    e = _err()
    if lib.ref_load_matrix(os.fsencode(path), C.byref(m), C.byref(k), C.byref(z), None, None,
                           None, e, 1024):
        raise RefError(e.value.decode())
    rp = np.zeros(m.value + 1, np.uint32)
    ci = np.zeros(max(z.value, 1), np.uint32)
    v = np.zeros(max(z.value, 1), np.float32)
    if lib.ref_load_matrix(os.fsencode(path), C.byref(m), C.byref(k), C.byref(z),
                           rp.ctypes.data, ci.ctypes.data, v.ctypes.data, e, 1024):
        raise RefError(e.value.decode())
    return m.value, k.value, rp, ci[: z.value].copy(), v[: z.value].copy()


SIM_FIELDS = ("gld_transactions", "gst_transactions", "requested_load_bytes",
              "transferred_load_bytes", "requested_store_bytes", "transferred_store_bytes",
              "ld_row_ptr", "ld_col_ind", "ld_val", "ld_b", "ld_c", "shared_loads",
              "shared_stores")


def ref_sim_metrics(m, k, row_ptr, col_ind, vals, b, op="sum", variant="crc", cf=2):
    """The reference SIMT simulator's counters (simt.hpp:117-162) for one run."""
    kind = {"naive": 0, "crc": 1, "crc-cwm": 2}[variant]
    b = np.ascontiguousarray(b, np.float32)
    out = (C.c_ulonglong * 13)()
    e = _err()
    if _load_ref().ref_sim_metrics(m, k, len(col_ind), _nz(row_ptr, np.uint32),
                                   _nz(col_ind, np.uint32), _nz(vals, np.float32),
                                   _nz(b.reshape(-1), np.float32), b.shape[1], op.encode(), kind,
                                   cf, out, e, 1024):
        raise RefError(e.value.decode())
    return dict(zip(SIM_FIELDS, (int(x) for x in out)))
