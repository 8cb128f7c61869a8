"""B200-native GE-SpMM (arXiv 2007.03179): CSR x dense SpMM-like with fused
sum / mean / max / min reduce ops (+ argmax/argmin), hand-written sm_100a
kernels behind the C ABI in include/gespmm/gespmm.h.

The compute path is libgespmm.so only; there is no CPU fallback.
"""
from .api import (  # noqa: F401
    CsrMatrix, DeviceCsr, DenseMatrix, Error, ExecOptions, FaultMode, GraphGenSpec,
    KernelConfig, KernelKind, KernelVariant, Plan, ReduceOp, ThroughputReport, bench,
    check_config, check_dense_valid, checksum, device_info, from_coo, gen_powerlaw,
    gen_uniform_random, make_random_dense, native_spmm, native_spmm_arg, ops,
    randomize_values, reduce_op_by_name, select_variant, spmm, variant_by_name,
    save_csr_cache, read_csr_cache, load_matrix, to_coo, ValidationReport, validate,
    require_canonical, parse_matrix_market, release_workspace,
)
from ._lib import LIB_PATH, experimental_built, launch_count  # noqa: F401

__version__ = "0.1.0"
