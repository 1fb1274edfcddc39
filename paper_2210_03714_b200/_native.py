"""ctypes binding of the C ABI in include/pf_b200.h (the product path; no fallback).

Importing this module loads ``_lib/libpfb200.so``; if it is missing the import fails loudly --
there is no CPU path behind this package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(os.environ.get("PF_B200_LIB") or Path(__file__).resolve().parent / "_lib" / "libpfb200.so")  # A/B builds

c_double_p = C.POINTER(C.c_double)
c_int_p = C.POINTER(C.c_int)


class PfStatus(C.Structure):
    _fields_ = [("code", C.c_int), ("batch_index", C.c_int), ("shift_index", C.c_int), ("column", C.c_int),
                ("pivot_magnitude", C.c_double), ("scale", C.c_double)]


class PfMethod(C.Structure):
    _fields_ = [("n_terms", C.c_int), ("shifts", c_double_p), ("n_sets", C.c_int), ("weights", c_double_p),
                ("has_poly", C.c_int), ("poly", c_double_p), ("constant", c_double_p), ("form", C.c_int)]


class PfPairMethod(C.Structure):
    _fields_ = [("n_pairs", C.c_int), ("c2", c_double_p), ("cw", c_double_p), ("sw", c_double_p),
                ("a0", C.c_double), ("a1", C.c_double)]


PF_FLAG_ASYNC = 1
PF_FLAG_FORCE_PIVOT = 2
PF_FLAG_PER_SHIFT = 4  # no (c, -c) pair merging: the reference's per-shift rounding sequence
PF_FLAG_REFERENCE_ORDER = 8  # n <= 128: dense.cpp's exact operation order, bit-identical results
PF_MAX_TERMS = 16
PF_SMALL_N = 128

# (name, restype, argtypes) -- every symbol include/pf_b200.h declares
_VP = C.c_void_p
_I64 = C.c_int64
SIGNATURES = [
    ("pf_version", C.c_int, []),
    ("pf_error_string", C.c_char_p, [C.c_int]),
    ("pf_context_create", C.c_int, [C.c_int, C.POINTER(_VP)]),
    ("pf_context_destroy", C.c_int, [_VP]),
    ("pf_context_set_stream", C.c_int, [_VP, _VP]),
    ("pf_context_launch_count", C.c_int64, [_VP]),
    ("pf_context_set_profile", C.c_int, [_VP, _VP]),
    ("pf_context_set_sticky_status", C.c_int, [_VP, C.c_int]),
    ("pf_context_pending_error", C.c_int, [_VP]),
    ("pf_one_norm_batched", C.c_int, [_VP, C.c_int, C.c_int, _VP, _I64, _I64, _VP]),
    ("pf_eval_dense_batched", C.c_int, [_VP, C.POINTER(PfMethod), C.c_int, C.c_int, _VP, _I64, _I64,
                                        C.POINTER(_VP), _I64, _I64, C.c_int, C.POINTER(PfStatus)]),
    ("pf_expm_batched", C.c_int, [_VP, C.POINTER(PfMethod), C.c_double, C.c_int, C.c_int, _VP, _I64, _I64, _VP,
                                  _VP, _VP, _I64, _I64, C.c_int, C.POINTER(PfStatus)]),
    ("pf_expm_phi1_batched", C.c_int, [_VP, C.POINTER(PfMethod), C.c_double, C.c_int, C.c_int, _VP, _I64, _I64,
                                       _VP, _VP, _VP, _VP, _I64, _I64, C.c_int, C.POINTER(PfStatus)]),
    ("pf_cossin_batched", C.c_int, [_VP, C.POINTER(PfPairMethod), C.c_double, C.c_int, C.c_int, _VP, _I64, _I64,
                                    _VP, _VP, _VP, _VP, _I64, _I64, C.c_int, C.POINTER(PfStatus)]),
    ("pf_action_block", C.c_int, [_VP, C.POINTER(PfMethod), C.c_int, C.c_int, _VP, _I64, _VP, _I64, C.c_int, _VP,
                                  _I64, C.c_int, C.POINTER(PfStatus)]),
    ("pf_lu_factor_batched", C.c_int, [_VP, C.c_int, C.c_int, _VP, _I64, _I64, _VP, C.c_double, C.c_int,
                                       C.POINTER(PfStatus)]),
    ("pf_lu_solve_batched", C.c_int, [_VP, C.c_int, C.c_int, C.c_int, _VP, _I64, _I64, _VP, _VP, _I64, _I64]),
    ("pf_solve_shifted_batched", C.c_int, [_VP, C.c_int, C.c_int, _VP, _I64, _I64, C.c_double, _VP, _I64, _I64,
                                           C.c_int, C.POINTER(PfStatus)]),
    ("pf_eval_scaled_batched", C.c_int, [_VP, C.POINTER(PfMethod), C.c_double, C.c_int, C.c_int, _VP, _I64, _I64,
                                         _VP, _VP, C.POINTER(_VP), _I64, _I64, C.c_int, C.POINTER(PfStatus)]),
    ("pf_squarings_batched", C.c_int, [_VP, C.c_int, C.c_int, _VP, _I64, _I64, C.c_double, _VP]),
    ("pf_ordered_sum", C.c_int, [_VP, C.c_int, C.POINTER(_VP), _I64, _VP]),
    ("pf_square_chain", C.c_int, [_VP, C.c_int, C.c_int, _VP, _VP]),
    ("pf_phi1_doubling", C.c_int, [_VP, C.c_int, C.c_int, _VP, _VP, _VP]),
    ("pf_cossin_doubling", C.c_int, [_VP, C.c_int, C.c_int, _VP, _VP, _VP]),
    ("pf_action_create", C.c_int, [_VP, C.POINTER(PfMethod), C.c_int, _VP, _I64, C.c_int, C.POINTER(C.c_int), C.c_int,
                                   C.POINTER(PfStatus), C.POINTER(_VP)]),
    ("pf_action_apply", C.c_int, [_VP, _VP, _I64, C.c_int, _VP, _I64, C.c_int, _VP, C.POINTER(PfStatus)]),
    ("pf_action_term_count", C.c_int, [_VP]),
    ("pf_action_destroy", C.c_int, [_VP]),
    ("pf_probe_dmma_tflops", C.c_double, [C.c_int]),
    ("pf_device_alloc", C.c_int, [_VP, C.c_size_t, C.POINTER(_VP)]),
    ("pf_device_free", C.c_int, [_VP, _VP]),
    ("pf_copy_to_device", C.c_int, [_VP, _VP, _VP, C.c_size_t]),
    ("pf_copy_to_host", C.c_int, [_VP, _VP, _VP, C.c_size_t]),
    ("pf_gemm_batched", C.c_int, [_VP, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _VP, _I64, _I64, _VP, _I64,
                                  _I64, C.c_double, _VP, _I64, _I64, C.c_double]),
    ("pf_tridiag_matvec_batched", C.c_int, [_VP, C.c_int, C.c_int, _VP, _VP, _VP, _VP, _I64, _VP, _I64]),
    ("pf_thomas_solve_batched", C.c_int, [_VP, C.c_int, C.c_int, _VP, _VP, _VP, _VP, _I64, _VP, _I64,
                                          C.POINTER(PfStatus)]),
    ("pf_pentadiag_solve_batched", C.c_int, [_VP, C.c_int, C.c_int, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _VP, _I64,
                                             C.POINTER(PfStatus)]),
    ("pf_tridiag_action", C.c_int, [_VP, C.POINTER(PfMethod), C.c_int, C.c_int, _VP, _VP, _VP, _VP, _I64, C.c_int,
                                    _VP, _I64, C.c_int, C.POINTER(PfStatus)]),
    ("pf_context_create_multi", C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(_VP)]),
    ("pf_context_device_count", C.c_int, [_VP]),
    ("pf_context_uses_nccl", C.c_int, [_VP]),
    ("pf_eval_multi_gpu", C.c_int, [_VP, C.POINTER(PfMethod), C.c_double, C.c_int, C.c_int, _VP, _I64, _VP, _VP, _I64,
                                    C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(PfStatus)]),
]
SIGNATURES += [
    ("pf_tridiag_op_create", C.c_int, [_VP, C.POINTER(PfMethod), C.c_int, _VP, _VP, _VP, C.c_int,
                                       C.POINTER(PfStatus), C.POINTER(_VP)]),
    ("pf_tridiag_op_apply", C.c_int, [_VP, C.POINTER(PfMethod), _VP, _I64, C.c_int, _VP, _I64, C.POINTER(PfStatus)]),
    ("pf_tridiag_op_destroy", C.c_int, [_VP]),
    ("pf_tridiag_factor_create", C.c_int, [_VP, C.c_int, _VP, _VP, _VP, C.POINTER(PfStatus), C.POINTER(_VP)]),
    ("pf_tridiag_factor_solve", C.c_int, [_VP, C.c_int, _VP, _I64, _VP, _I64]),
    ("pf_tridiag_factor_destroy", C.c_int, [_VP]),
    ("pf_add_identity_rows", C.c_int, [_VP, C.c_int, C.c_int, C.c_int, _VP, _I64, _VP, _I64]),
    ("pf_sum_diff", C.c_int, [_VP, _I64, _VP, _VP, _VP, _VP]),
]
PF_REC_NONE, PF_REC_EXP, PF_REC_EXP_PHI1 = 0, 1, 2


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    p = Path(path) if path else _LIB_PATH
    if not p.exists():
        raise ImportError("paper_2210_03714_b200: native engine %s is missing; run "
                          "`python -m paper_2210_03714_b200.build` (there is no CPU fallback)" % p)
    lib = C.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()
