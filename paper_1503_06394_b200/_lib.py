"""ctypes binding of libchebld.so (include/cheb_logdet.h).  Argument marshalling
only: every step of the path runs in the library's CUDA kernels.  There is no
CPU fallback -- if the library is missing this module raises at import.
"""
import ctypes
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SO_PATH = os.environ.get("CHEB_LIB") or os.path.join(PKG, "libchebld.so")  # CHEB_LIB: tuning builds
HEADER = os.path.join(ROOT, "include", "cheb_logdet.h")

CL_OK, CL_EINVAL, CL_EDIM, CL_ENOMEM, CL_ECUDA, CL_ENONFINITE = 0, -1, -2, -3, -4, -5
OP_KIND = {"csr": 0, "rank1": 1, "btb": 2, "family": 3}


class ChebError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class CLCsr(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class CLOperator(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("A", CLCsr), ("At", CLCsr),
                ("r1_c", ctypes.c_double), ("r1_u", ctypes.c_void_p)]


class CLSpectrum(ctypes.Structure):
    _fields_ = [("lambda_min", ctypes.c_double), ("lambda_max", ctypes.c_double),
                ("res_min", ctypes.c_double), ("res_max", ctypes.c_double),
                ("a", ctypes.c_double), ("b", ctypes.c_double),
                ("hi_bound", ctypes.c_double), ("lanczos_steps", ctypes.c_int32), ("num_probes", ctypes.c_int32)]


class CLResult(ctypes.Structure):
    _fields_ = [("logdet", ctypes.c_double), ("stderr_", ctypes.c_double),
                ("num_probes", ctypes.c_int64), ("degree", ctypes.c_int32),
                ("probe_block", ctypes.c_int32), ("per_probe", ctypes.c_void_p),
                ("moments", ctypes.c_void_p), ("elapsed_s", ctypes.c_double)]


def header_symbols():
    """Names of the functions include/cheb_logdet.h declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|int64_t|const char \*)\s*\**\s*(cheb_\w+)\s*\(",
                                 txt, flags=re.M)))


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(SO_PATH)
    I, I32, I64, U64, D, P, SZ = (ctypes.c_int, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                  ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t)
    OPP = ctypes.POINTER(CLOperator)
    sig = {
        "cheb_coeffs_log": (I, [D, D, I32, P]),
        "cheb_workspace_bytes": (SZ, [OPP, I32]),
        "cheb_moments": (I, [OPP, D, D, I32, I64, I64, U64, I32, P, SZ, P, P]),
        "cheb_finalize": (I, [P, P, I64, I32, P, P, P]),
        "cheb_power_moments": (I, [OPP, D, I32, I64, I64, U64, I32, P, SZ, P, P]),
        "cheb_taylor_coeffs": (I, [D, I32, P]),
        "cheb_affine_power_moments": (I, [OPP, D, D, I32, I64, I64, U64, I32, P, SZ, P, P]),
        "cheb_norm_bound": (I, [OPP, P, P]),
        "cheb_quadform": (I, [ctypes.POINTER(CLCsr), P, P, P]),
        "cheb_gershgorin": (I, [ctypes.POINTER(CLCsr), P, P]),
        "cheb_quadform_split": (I, [ctypes.POINTER(CLCsr), P, P, P]),
        "cheb_family_gershgorin": (I, [ctypes.POINTER(CLCsr), I32, P, P, P]),
        "cheb_family_moments": (I, [ctypes.POINTER(CLCsr), I32, P, P, I32, I64, I64, U64, I32, P, SZ, P, P]),
        "cheb_logdet": (I, [OPP, D, D, I32, I32, U64, I32, ctypes.POINTER(CLResult)]),
        "cheb_logdet_host": (I, [OPP, D, D, I32, I32, U64, I32, ctypes.POINTER(CLResult)]),
        "cheb_moments_host": (I, [OPP, D, D, I32, I64, I64, U64, I32, P]),
        "cheb_spectrum_bounds": (I, [OPP, I32, I32, U64, ctypes.POINTER(CLSpectrum), P]),
        "cheb_bounds_btb": (I, [OPP, P, P]),
        "cheb_probes": (I, [I64, U64, I64, I32, P, P]),
        "cheb_launch_count": (I64, []),
        "cheb_profile_begin": (I, []),
        "cheb_profile_end": (I, [ctypes.POINTER(D), ctypes.POINTER(I64)]),
        "cheb_profile_spmm": (I, [ctypes.POINTER(D), ctypes.POINTER(I64)]),
        "cheb_workspace_status": (I, [P, ctypes.POINTER(ctypes.c_uint32), P]),
        "cheb_profile_persistent": (I, [ctypes.POINTER(D), ctypes.POINTER(I64)]),
        "cheb_set_persistent": (I, [I32]),
        "cheb_set_small_tiles": (I, [I32]),
        "cheb_get_small_tiles": (I, []),
        "cheb_set_doubling": (I, [I32]),
        "cheb_get_doubling": (I, []),
        "cheb_set_resident": (I, [I32]),
        "cheb_get_resident": (I, []),
        "cheb_last_schedule": (I, []),
        "cheb_release_cache": (I, []),
        "cheb_last_error": (ctypes.c_char_p, []),
        "cheb_version": (I, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc):
    if rc != CL_OK:
        raise ChebError(rc, load().cheb_last_error().decode())
    return rc
