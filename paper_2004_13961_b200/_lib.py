"""ctypes binding of the C ABI in include/legpcg_b200.h.

The library is built in-tree (``__graft_entry__.build()`` or
``make -C paper_2004_13961_b200/csrc``).  There is no CPU fallback: every
compute entry point of this package goes through this library and raises if
it is missing or no sm_100 GPU is present.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_PATH = os.environ.get("LP_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "liblegpcg_b200.so")

LP_OK = 0
LP_ERR_CUDA = -1
LP_ERR_ARG = -2
LP_ERR_NONPOSITIVE = -3
LP_ERR_ZERO_PIVOT = -4
LP_ERR_INDEFINITE = -5
LP_ERR_NODEVICE = -6
LP_ERR_OOM = -7

_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_dbl = ctypes.c_double


class LpReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("converged", ctypes.c_int32),
                ("pad_", ctypes.c_int32), ("final_relative_residual", ctypes.c_double),
                ("loop_seconds", ctypes.c_double), ("indefinite_value", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64)]


_SIGS = {
    "lp_last_error": (ctypes.c_char_p, []),
    "lp_version": (ctypes.c_char_p, []),
    "lp_kernel_launches": (_i64, []),
    "lp_init": (_i32, [_i32]),
    "lp_plan_create": (_i32, [_i32, _vp, _vp, ctypes.POINTER(_vp)]),
    "lp_plan_destroy": (_i32, [_vp]),
    "lp_plan_table": (_i32, [_vp, _vp]),
    "lp_tensor_bdlt": (_i32, [_vp, _i32, _vp, _vp, _vp]),
    "lp_tensor_fdlt": (_i32, [_vp, _i32, _vp, _vp, _vp]),
    "lp_operator_create": (_i32, [_vp, _i32, _vp, _i32, ctypes.POINTER(_vp), _vp,
                                  ctypes.POINTER(_vp)]),
    "lp_operator_destroy": (_i32, [_vp]),
    "lp_apply": (_i32, [_vp, _i32, _vp, _vp, _vp]),
    "lp_apply_dot": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp]),
    "lp_csr_create": (_i32, [_i64, _i64, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "lp_box_assemble": (_i32, [_i32, _i32, _i32, _vp, _vp, ctypes.POINTER(_vp), _i32, _vp,
                               ctypes.POINTER(_vp)]),
    "lp_blocks_1d": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp]),
    "lp_mass_contract": (_i32, [_i32, _i32, _vp, _vp, _vp]),
    "lp_matrix_nnz": (_i32, [_vp, ctypes.POINTER(_i64)]),
    "lp_matrix_export": (_i32, [_vp, _i32, _vp, _vp, _vp]),
    "lp_ilu0": (_i32, [_vp, _dbl, ctypes.POINTER(_i64), _vp]),
    "lp_ilu0_ranks": (_i32, [_vp, _i32, _vp, _dbl, ctypes.POINTER(_i64), _vp]),
    "lp_ilu0_rank": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _dbl, ctypes.POINTER(_i64), _vp]),
    "lp_ilu_rank_arrays": (_i32, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp, _vp]),
    "lp_ilu0_rank_prepare": (_i32, [_vp, ctypes.POINTER(_i64), _vp]),
    "lp_forward_sub": (_i32, [_vp, _vp, _vp, _vp]),
    "lp_backward_sub": (_i32, [_vp, _vp, _vp, _vp]),
    "lp_precond_apply": (_i32, [_vp, _vp, _vp, _vp]),
    "lp_precond_apply_rz": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "lp_spmv": (_i32, [_vp, _vp, _vp, _vp]),
    "lp_ilu_destroy": (_i32, [_vp]),
    "lp_pcg_solve": (_i32, [_vp, _vp, _vp, _vp, _i32, _dbl, _i64, _vp,
                            ctypes.POINTER(LpReport), _vp]),
    "lp_dot": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "lp_copy2d": (_i32, [_i64, _i32, _vp, _i64, _vp, _i64, _vp]),
    "lp_sweep_ranks": (_i32, [_vp, _i32, _vp, _i32, _vp, _i32, _vp, _vp]),
    "lp_sweep_rank": (_i32, [_vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "lp_sweep_prefill": (_i32, [_i64, _vp, _vp]),
    "lp_ipc_alloc": (_i32, [_i64, ctypes.POINTER(_vp), _vp]),
    "lp_ipc_free": (_i32, [_vp]),
    "lp_ipc_open": (_i32, [_vp, ctypes.POINTER(_vp)]),
    "lp_ipc_close": (_i32, [_vp]),
    "lp_update_p": (_i32, [_i64, _vp, _vp, _dbl, _i32, _vp]),
    "lp_update_xr": (_i32, [_i64, _vp, _vp, _vp, _vp, _dbl, _vp, _vp]),
    "lp_slab_forward": (_i32, [_vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "lp_slab_middle": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "lp_comm_init": (_i32, [_vp, _i32, _i32, _i32, ctypes.POINTER(_vp)]),
    "lp_comm_destroy": (_i32, [_vp]),
    "lp_comm_allreduce_dd": (_i32, [_vp, _vp, _vp]),
    "lp_comm_dot": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp]),
    "lp_comm_alltoall": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "lp_slab_backward": (_i32, [_vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None
_initialised = False


def load(init_device=True):
    """Load the library (and bind the current torch device) or raise."""
    global _lib, _initialised
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"CUDA library not built: {LIB_PATH} is missing "
                    "(run __graft_entry__.build()); there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        if init_device and not _initialised:
            import torch
            if not torch.cuda.is_available():
                raise RuntimeError("legpcg_b200 requires an sm_100 (B200) GPU; none is visible")
            rc = _lib.lp_init(torch.cuda.current_device())
            if rc != LP_OK:
                raise RuntimeError(last_error())
            _initialised = True
    return _lib


def last_error():
    return (_lib.lp_last_error() or b"").decode()


def check(rc, what=""):
    """Map an LP_ERR_* code to the reference's exception types."""
    if rc == LP_OK:
        return
    msg = last_error()
    if rc in (LP_ERR_ARG, LP_ERR_NONPOSITIVE):
        raise ValueError(msg)
    if rc == LP_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def stream_ptr():
    import torch
    return torch.cuda.current_stream().cuda_stream
