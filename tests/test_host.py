"""CPU: the C-ABI library loads and exports every declared symbol; host logic
(generators, checksum, lookups, argument checks that fire before any device
work) matches the reference.  No compute calls here — they need a GPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2007_03179_b200 as G
from paper_2007_03179_b200 import _lib
from conftest import ROOT


def _header_functions():
    text = open(os.path.join(ROOT, "include", "gespmm", "gespmm.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gespmm_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    declared = _header_functions()
    assert len(declared) >= 20
    assert sorted(declared) == sorted(_lib.EXPORTS)
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                        text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", nm, re.M), f"{name} not exported with C linkage"


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_defaults():
    assert _lib.lib().gespmm_abi_version() == 2
    o = _lib.default_options()
    assert (o.variant, o.cf, o.exact, o.arg_kind, o.validate, o.l2_hints) == (0, 2, 1, 0, 1, 1)


def test_generator_pins(golden):
    for pin in golden["generator"]:
        if pin["kind"] == "gen_uniform":
            a = G.gen_uniform_random(G.GraphGenSpec(pin["rows"], pin["nnz"], pin["seed"],
                                                    pin["loops"]))
            h = _fnv(a.row_ptr, a.col_ind, a.vals)
        elif pin["kind"] == "randomize_values":
            m = G.CsrMatrix(1, 1, np.zeros(2, np.uint32), np.zeros(pin["nnz"], np.uint32),
                            np.ones(pin["nnz"], np.float32))
            G.randomize_values(m, pin["seed"])
            h = _fnv(m.vals)
        else:
            d = G.make_random_dense(pin["rows"], pin["cols"], pin["seed"])
            assert G.checksum(d) == pin["checksum"]
            continue
        assert h == pin["fnv"], pin


def _fnv(*arrays):
    h = 1469598103934665603
    for a in arrays:
        for byte in np.ascontiguousarray(a).tobytes():
            h = ((h ^ byte) * 1099511628211) & ((1 << 64) - 1)
    return h


def test_generator_errors():
    with pytest.raises(G.Error, match="feasible"):
        G.gen_uniform_random(G.GraphGenSpec(4, 20, 0, False))
    G.gen_uniform_random(G.GraphGenSpec(4, 16, 0, True))
    with pytest.raises(G.Error, match="zero rows"):
        G.gen_uniform_random(G.GraphGenSpec(0, 3, 0))


def test_generator_reference_shape_mean_degree():
    m = G.gen_uniform_random(G.GraphGenSpec(65536, 655360, 1))
    assert m.nnz() == 655360 and m.mean_degree() == 10.0
    deg = np.diff(m.row_ptr.astype(np.int64))
    assert deg.max() < 64


def test_powerlaw_generator_shape_and_determinism():
    a = G.gen_powerlaw(20000, 1_000_000, 4000, 1.0, 3, threads=1)
    b = G.gen_powerlaw(20000, 1_000_000, 4000, 1.0, 3, threads=7)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_ind, b.col_ind)
    assert a.nnz() == 1_000_000
    deg = np.diff(a.row_ptr.astype(np.int64))
    assert deg.max() == 4000
    assert np.median(deg) < deg.mean()  # skewed
    # canonical: strictly increasing columns, no self loops
    rows = np.repeat(np.arange(20000), deg)
    assert np.all(a.col_ind != rows)
    same_row = rows[1:] == rows[:-1]
    assert np.all(a.col_ind[1:][same_row] > a.col_ind[:-1][same_row])
    # in-degree also heavy tailed (columns drawn from the same weights)
    indeg = np.bincount(a.col_ind, minlength=20000)
    assert indeg.max() > 10 * indeg.mean()
    c = G.gen_powerlaw(20000, 1_000_000, 4000, 1.0, 4)
    assert not np.array_equal(a.col_ind, c.col_ind)


def test_select_variant_matches_reference_rule():
    for n in range(1, 2049):
        v = G.select_variant(n)
        if n <= 32:
            assert v == G.KernelVariant.crc()
        else:
            assert v == G.KernelVariant.crc_cwm(2)


def test_reduce_ops_laws_and_seeds():
    """test_reduce_op.cpp:24-46, with min/mean added deliberately (the reference
    pins "min" as unknown; this framework defines it)."""
    rng = np.random.default_rng(2024)
    for op in (G.ops.sum(), G.ops.max(), G.ops.min()):
        for _ in range(2000):
            a, b, c = (float(x) for x in rng.integers(-4096, 4097, 3))
            assert op.fold(op.fold(a, b), c) == op.fold(a, op.fold(b, c))
            assert op.fold(a, b) == op.fold(b, a)
            assert op.fold(op.init, a) == a
    assert G.ops.sum().init == 0.0
    assert G.ops.max().init == float(np.finfo(np.float32).min)
    assert G.ops.min().init == float(np.finfo(np.float32).max)
    assert G.reduce_op_by_name("sum").name == "sum"
    assert G.reduce_op_by_name("min").name == "min"
    assert G.reduce_op_by_name("mean").name == "mean"
    with pytest.raises(G.Error, match="unknown reduce op"):
        G.reduce_op_by_name("median")


def test_kernel_config_validation():
    """test_kernel_spec.cpp:89-98."""
    for bad in (G.KernelConfig(33, 8, G.KernelVariant.crc()),
                G.KernelConfig(2, 8, G.KernelVariant.crc()),
                G.KernelConfig(32, 0, G.KernelVariant.crc()),
                G.KernelConfig(32, 8, G.KernelVariant.crc_cwm(3)),
                G.KernelConfig(32, 8, G.KernelVariant.crc_cwm(16))):
        with pytest.raises(G.Error):
            G.check_config(bad)
    G.check_config(G.KernelConfig(32, 8, G.KernelVariant.crc_cwm(8)))
    G.check_config(G.KernelConfig(64, 1, G.KernelVariant.naive()))
    assert G.variant_by_name("crc-cwm", 4) == G.KernelVariant.crc_cwm(4)
    with pytest.raises(G.Error):
        G.variant_by_name("fast")


def test_from_coo_canonicalises():
    m = G.from_coo(2, 2, [(0, 1, 2.0), (1, 0, 3.0)])
    assert m.row_ptr.tolist() == [0, 1, 2] and m.col_ind.tolist() == [1, 0]
    m = G.from_coo(3, 3, [])
    assert m.row_ptr.tolist() == [0, 0, 0, 0]
    m = G.from_coo(1, 1, [(0, 0, 1.0), (0, 0, 2.0)])
    assert m.vals.tolist() == [3.0]
    m = G.from_coo(1, 1, [(0, 0, 1.0), (0, 0, 2.0)], policy="last")
    assert m.vals.tolist() == [2.0]
    with pytest.raises(G.Error, match="outside declared"):
        G.from_coo(2, 2, [(3, 1, 1.0)])


def test_host_checks_before_any_device_work(golden):
    """Dimension and length errors are raised on the host with the reference's text."""
    for case in golden["validation"]:
        if case["name"] not in ("dimension_mismatch", "col_vals_length_mismatch",
                                "row_ptr_wrong_length"):
            continue
        a = G.CsrMatrix(case["m"], case["k"], np.array(case["row_ptr"], np.uint32),
                        np.array(case["col_ind"], np.uint32), np.array(case["vals"], np.float32))
        b = G.DenseMatrix.zeros(case["b_rows"], case["n"])
        with pytest.raises(G.Error) as ei:
            G.native_spmm(a, b, G.select_variant(case["n"]), G.ops.sum())
        assert str(ei.value) == case["error"]


def test_int32_arg_range_is_checked_before_device_work():
    """arg is int32 in the C ABI: a max/min call whose CSR positions (edge
    args) or columns (column args) would not fit is refused with EINVAL before
    any device work, instead of writing wrapped indices."""
    L = _lib.lib()
    big = (1 << 31) + 5
    csr = _lib.Csr(4, 8, big, None, None, None)       # never dereferenced
    arg = ctypes.c_void_p(16)                          # never written
    for entry in ("gespmm_spmm_device", "gespmm_spmm_host"):
        o = _lib.default_options(validate=0)
        if entry == "gespmm_spmm_device":
            st = L.gespmm_spmm_device(ctypes.byref(csr), None, 4, _lib.MAX, None, arg,
                                      ctypes.byref(o), None)
        else:
            st = L.gespmm_spmm_host(ctypes.byref(csr), None, 8, 4, _lib.MAX, None, arg,
                                    ctypes.byref(o))
        assert st == _lib.EINVAL
        msg = L.gespmm_last_error().decode()
        assert "do not fit the int32 arg" in msg and "arg_kind = column" in msg, msg
    wide = _lib.Csr(4, (1 << 32) - 1, 10, None, None, None)
    o = _lib.default_options(validate=0, arg_kind=_lib.ARG_COLUMN)
    st = L.gespmm_spmm_device(ctypes.byref(wide), None, 4, _lib.MAX, None, arg, ctypes.byref(o), None)
    assert st == _lib.EINVAL and "column indices" in L.gespmm_last_error().decode()
