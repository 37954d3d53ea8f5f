"""ctypes loader for libslb.so (the C-ABI in include/slb.h).  No fallback: if the
library is missing or fails to load, every entry point raises."""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libslb.so")
_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
D = ctypes.c_double


class SlbError(RuntimeError):
    pass


class OperatorDesc(ctypes.Structure):
    _fields_ = [("kernel", I32), ("ns", I32), ("nt", I32), ("ms", I32), ("mt", I32),
                ("n_panels_global", I64), ("panel_begin", I64), ("panel_end", I64),
                ("n_trg_local", I64), ("n_on_local", I64), ("c_identity", D),
                ("x_trg", P), ("y_fine", P), ("n_fine", P), ("w_fine", P), ("eta_fine", P),
                ("eta", D), ("row_ptr", P), ("panel_idx", P), ("blocks", P), ("blocks_folded", I32),
                ("n_bodies_local", I64), ("body_of_panel_local", P), ("y_coarse", P), ("w_coarse", P),
                ("panel_nt", P), ("panel_mt", P), ("panel_ns", P), ("panel_ms", P)]


_SIGS = {
    "slb_abi_version": (I32, []),
    "slb_last_error": (ctypes.c_char_p, []),
    "slb_eta_cfie": (D, [D]),
    "slb_coincident_count": (ctypes.c_longlong, []),
    "slb_coincident_reset": (None, []),
    "slb_launch_count": (ctypes.c_ulonglong, []),
    "slb_upsample": (I32, [I64, I32, I32, I32, I32, I32, P, P, P]),
    "slb_upsample_ragged": (I32, [I64, P, P, P, P, I32, P, P, P]),
    "slb_farfield_laplace_dl": (I32, [I64, P, I64, P, P, P, P, P, P]),
    "slb_farfield_stokes_sldl": (I32, [I64, P, I64, P, P, P, P, D, P, P, P]),
    "slb_nearcorr_apply": (I32, [I64, I32, I32, I32, P, P, P, P, P, P]),
    "slb_nearcorr_fold": (I32, [I32, I64, P, P, P, I32, I32, I32, I32, P, P, P, P, D, P, P]),
    "slb_fill_blocks": (I32, [ctypes.c_uint64, ctypes.c_uint64, I64, D, P, P]),
    "slb_nearcorr_quad": (I32, [I32, I64, P, P, P, P, I32, I32, P, P, I32, D, P, P]),
    "slb_nearcorr_quad_ragged": (I32, [I32, I64, P, P, P, P, I64, P, P, P, P, I32, D, P, P]),
    "slb_near_build": (I32, [I64, P, I64, I32, P, P, P, P, P, I64, ctypes.POINTER(I64), P]),
    "slb_comm_unique_id": (I32, [P]),
    "slb_comm_create": (I32, [P, I32, I32, ctypes.POINTER(P)]),
    "slb_comm_destroy": (I32, [P]),
    "slb_comm_collective_counts": (I32, [P, ctypes.POINTER(ctypes.c_longlong)]),
    "slb_operator_create": (I32, [ctypes.POINTER(OperatorDesc), P, ctypes.POINTER(P)]),
    "slb_matvec": (I32, [P, P, P, P]),
    "slb_matvec_host": (I32, [P, P, P, P]),
    "slb_operator_last_timings": (I32, [P, ctypes.POINTER(ctypes.c_float)]),
    "slb_operator_prepare": (I32, [P, P, P]),
    "slb_operator_launches_per_matvec": (I32, [P]),
    "slb_operator_nvls": (I32, [P]),
    "slb_nvls_supported": (I32, []),
    "slb_operator_destroy": (I32, [P]),
    "slb_gmres": (I32, [P, P, P, I32, I32, D, ctypes.POINTER(I32), ctypes.POINTER(D), P]),
    "slb_mobility_solve": (I32, [P, P, P, P, P, I32, I32, D, ctypes.POINTER(I32), ctypes.POINTER(D), P]),
    "slb_bench_dfma": (I32, [I64, ctypes.POINTER(D), P]),
}

# symbols declared in include/slb.h (checked by the CPU test that loads the library)
DECLARED = list(_SIGS)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise SlbError(f"libslb.so not built ({SO_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(SO_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


STATUS = {0: "SLB_OK", 1: "SLB_ERR_INVALID_ARG", 2: "SLB_ERR_CUDA", 3: "SLB_ERR_NCCL", 4: "SLB_ERR_OOM",
          5: "SLB_ERR_UNSUPPORTED"}


def check(status):
    if status != 0:
        msg = lib().slb_last_error().decode(errors="replace")
        raise SlbError(f"{STATUS.get(status, status)}: {msg}")
