"""ctypes binding of libpdcs.so (include/pdcs.h).

The shared library is built in-tree by `build_native()` (nvcc, sm_100a).
There is no fallback: if the library or a CUDA device is missing, every
device entry point raises `NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpdcs.so")
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]

# cone kinds / scale modes / stop reasons (pdcs.h)
FREE, ZERO, NONNEG, SOC, EXP, DUAL_EXP = range(6)
SCALE_NONE, SCALE_DIRECT, SCALE_INVERT = range(3)
STOP_NONE, STOP_CHECK, STOP_MAXITER, STOP_BATCH, STOP_PRINT, STOP_ERROR = range(6)
NMET, NRAY = 20, 9
(MET_RV2, MET_RVMAX, MET_HMAX, MET_GXMAX, MET_RPMAX, MET_YH, MET_H1, MET_V1SQ, MET_V1MAX,
 MET_V2SQ, MET_V2MAX, MET_CMAX, MET_GTYMAX, MET_CX, MET_LSUM, MET_USUM, MET_C1,
 MET_NONFINITE, MET_XX, MET_YY) = range(20)


class NativeUnavailable(RuntimeError):
    """libpdcs.so could not be loaded or no CUDA device is present."""


class NativeError(RuntimeError):
    """A libpdcs entry point returned a non-zero status."""


class PdcsBlock(C.Structure):
    _fields_ = [("kind", C.c_int32), ("start", C.c_int32), ("dim", C.c_int32), ("smode", C.c_int32)]


_I64 = ["k_bar", "k", "trials", "k_bar_stop", "max_iter", "check_freq", "print_freq",
        "stop", "reason", "error", "new_iter", "accepted", "pending", "adaptive", "use_fixed_beta",
        "n_trials_total", "n_accepted_total", "nan_after", "n_primal_proj", "spare0"]
_F64 = ["eta_hat", "eta_try", "eta", "omega", "beta", "W", "fixed_beta", "tau", "sigma",
        "pa", "pb", "pbeta", "peta", "pW", "c1", "h1",
        "movement", "interaction", "eta_bar", "p_obj", "d_obj", "max_err"]


class PdcsCtrl(C.Structure):
    _fields_ = [(f, C.c_int64) for f in _I64] + [(f, C.c_double) for f in _F64] + [
        ("spare", C.c_double * 4)]


_P = C.c_void_p
_DESC_PTRS = [
    "d_g_rowptr", "d_g_colidx", "d_g_val", "d_gt_rowptr", "d_gt_colidx", "d_gt_val", "d_perm",
    "d_g_val0", "d_c", "d_h", "d_l", "d_u", "d_c0", "d_h0", "d_l0", "d_u0", "d_d1", "d_d2",
    "d_x", "d_y", "d_xh", "d_yh", "d_xb", "d_yb", "d_xa", "d_ya", "d_xpa", "d_ypa",
    "d_gx", "d_gty", "d_gxa", "d_gtya", "d_w", "d_gxh", "d_gth", "d_gtr", "d_xt",
    "d_tx0", "d_tx1", "d_tx2", "d_ty0", "d_ty1", "d_ty2",
]


class PdcsEngineDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("m", C.c_int32), ("num_box", C.c_int32), ("nnz", C.c_int32),
        ("m_zero", C.c_int32), ("m_elem", C.c_int32), ("n_pcones", C.c_int32), ("n_dcones", C.c_int32),
        ("h_pcone_kind", C.POINTER(C.c_int32)), ("h_pcone_dim", C.POINTER(C.c_int32)),
        ("h_dcone_kind", C.POINTER(C.c_int32)), ("h_dcone_dim", C.POINTER(C.c_int32)),
        ("allow_nonuniform_dual_soc", C.c_int32), ("pad0", C.c_int32),
    ] + [(p, _P) for p in _DESC_PTRS]


_SIGS = {
    "pdcs_last_error": (C.c_char_p, []),
    "pdcs_abi_version": (C.c_int, []),
    "pdcs_launch_count": (C.c_int64, []),
    "pdcs_spmv_csr": (C.c_int, [C.c_int32, _P, _P, _P, _P, _P, _P]),
    "pdcs_transpose_csr": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pdcs_project_segments": (C.c_int, [C.c_int32, _P, _P, C.POINTER(PdcsBlock), C.c_int32, _P,
                                        C.POINTER(C.c_int32), _P]),
    "pdcs_project_segments_ex": (C.c_int, [C.c_int32, _P, _P, C.POINTER(PdcsBlock), C.c_int32, _P,
                                           C.c_double, C.c_int32, C.POINTER(C.c_int32), _P]),
    "pdcs_project_box": (C.c_int, [C.c_int32, _P, _P, _P, _P, _P]),
    "pdcs_vec_axpby": (C.c_int, [C.c_int32, C.c_double, _P, C.c_double, _P, C.c_double, _P, _P]),
    "pdcs_engine_create": (C.c_int, [C.POINTER(PdcsEngineDesc), _P, C.POINTER(_P)]),
    "pdcs_engine_destroy": (None, [_P]),
    "pdcs_precondition": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32]),
    "pdcs_stats": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "pdcs_engine_info": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "pdcs_engine_get_ctrl": (C.c_int, [_P, C.POINTER(PdcsCtrl)]),
    "pdcs_engine_set_ctrl": (C.c_int, [_P, C.POINTER(PdcsCtrl)]),
    "pdcs_run_inner": (C.c_int, [_P, C.c_int32]),
    "pdcs_batch_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, _P, C.POINTER(C.c_void_p)]),
    "pdcs_batch_run": (C.c_int, [_P, C.c_int32]),
    "pdcs_batch_destroy": (None, [_P]),
    "pdcs_flush": (C.c_int, [_P]),
    "pdcs_profile_slot": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_char_p), C.c_int32]),
    "pdcs_engine_spmv": (C.c_int, [_P, C.c_int32, _P, _P]),
    "pdcs_metrics": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, C.POINTER(C.c_double)]),
    "pdcs_rays": (C.c_int, [_P, _P, _P, _P, _P, C.c_double, C.c_double, C.POINTER(C.c_double)]),
    "pdcs_gap_probe": (C.c_int, [_P, _P, _P, _P, _P, C.c_double, C.c_double, C.c_double,
                                 C.POINTER(C.c_double)]),
    "pdcs_gap_probes": (C.c_int, [_P, _P, _P, _P, _P, C.POINTER(C.c_double), C.c_int32, C.c_double,
                                  C.c_double, C.POINTER(C.c_double)]),
    "pdcs_dist2": (C.c_int, [_P, C.c_int32, _P, _P, C.POINTER(C.c_double)]),
    "pdcs_dot_diff": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, C.POINTER(C.c_double)]),
    "pdcs_project_set": (C.c_int, [_P, C.c_int32, _P, _P]),
    "pdcs_project_set_ex": (C.c_int, [_P, C.c_int32, _P, _P, C.c_double, C.c_int32]),
    "pdcs_step_input": (C.c_int, [_P, C.c_int32, _P, _P, C.c_double, _P]),
    "pdcs_axpby": (C.c_int, [_P, C.c_int32, C.c_double, _P, C.c_double, _P, _P]),
    "pdcs_unscale": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pdcs_debug_inject_nan": (C.c_int, [_P, C.c_int64]),
    "pdcs_comm_unique_id": (C.c_int, [C.c_char_p]),
    "pdcs_engine_set_uniform_box": (C.c_int, [_P, C.c_double, C.c_double]),
    "pdcs_engine_set_persist": (C.c_int, [_P, C.c_int32]),
    "pdcs_engine_set_comm": (C.c_int, [_P, C.c_char_p, C.c_int32, C.c_int32]),
    "pdcs_engine_set_xsplit": (C.c_int, [_P, C.POINTER(C.c_int32), C.c_int32]),
    "pdcs_allgather_x": (C.c_int, [_P, C.POINTER(C.c_void_p), C.c_int32]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def build_native(force: bool = False, verbose: bool = False) -> str:
    """Compile libpdcs.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))]
    newest = max(os.path.getmtime(s) for s in srcs + [os.path.join(INCLUDE, "pdcs.h")])
    if not force and os.path.exists(LIB_PATH):
        if os.path.getmtime(LIB_PATH) >= newest:
            return LIB_PATH
    cmd = ["nvcc", *NVCC_FLAGS, "-I", INCLUDE, "-o", LIB_PATH + ".tmp",
           os.path.join(CSRC, "pdcs_engine.cu"), "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        print(res.stderr)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    # stamp the library with the sources' time at build start: a source edited
    # while nvcc ran is then newer and triggers the next rebuild
    os.utime(LIB_PATH, (newest, newest))
    return LIB_PATH


def load_library() -> C.CDLL:
    """Load libpdcs.so and declare its signatures (no CUDA device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing; build it with paper_2603_15504_b200._native.build_native()")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib() -> C.CDLL:
    """The loaded library, after checking that a CUDA device is usable."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("paper_2603_15504_b200 needs a CUDA device (B200, sm_100a); none is available")
    return load_library()


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = _lib.pdcs_last_error().decode() if _lib is not None else "unknown"
        raise NativeError(f"{what} failed (status {rc}): {msg}")


def launch_count() -> int:
    return int(load_library().pdcs_launch_count())
