"""ctypes binding of libzeus_sm100.so (include/zeus_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every compute entry point raises ``ZeusNativeError``.
"""

from __future__ import annotations

import ctypes
import os

__all__ = ["ZeusNativeError", "lib", "check", "LIB_PATH", "BfgsParams", "BfgsOut",
           "OBJ_ROSENBROCK", "OBJ_RASTRIGIN", "OBJ_ACKLEY", "OBJ_GOLDSTEIN_PRICE",
           "EXPORTED_SYMBOLS"]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZEUS_LIB") or os.path.join(HERE, "libzeus_sm100.so")

OBJ_ROSENBROCK = 0
OBJ_RASTRIGIN = 1
OBJ_ACKLEY = 2
OBJ_GOLDSTEIN_PRICE = 3

ABI_VERSION = 2

_i32, _i64, _u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
_int, _dbl, _vp, _sz = ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t


class ZeusNativeError(RuntimeError):
    """The CUDA library is unavailable or a device call failed."""


class BfgsParams(ctypes.Structure):
    _fields_ = [("theta", _dbl), ("iter_bfgs", _i32), ("iter_ls", _i32),
                ("c1_armijo", _dbl), ("alpha0", _dbl), ("shrink", _dbl)]


class BfgsOut(ctypes.Structure):
    _fields_ = [("x_final", _vp), ("ld_out", _i64), ("f_final", _vp), ("grad_norm", _vp),
                ("iterations", _vp), ("status", _vp), ("ls_trials", _vp),
                ("grad_evals", _vp), ("rows", _vp), ("ld_rows", _i64), ("irows", _vp)]


# name -> (restype, argtypes); every symbol declared in include/zeus_b200.h
_SIGNATURES = {
    "zeus_abi_version": (_int, []),
    "zeus_last_error": (ctypes.c_char_p, []),
    "zeus_sm_count": (_int, [_int]),
    "zeus_philox_uniform": (_int, [_u64, _i64, _i64, _u64, _i64, _dbl, _dbl, _vp, _vp]),
    "zeus_objective_value": (_int, [_int, _int, _i64, _vp, _i64, _vp, _vp]),
    "zeus_objective_gradient": (_int, [_int, _int, _i64, _vp, _i64, _vp, _vp, _vp]),
    "zeus_pso_workspace_bytes": (_sz, [_i64]),
    "zeus_pso_init": (_int, [_int, _int, _i64, _i64, _u64, _dbl, _dbl, _vp, _vp, _vp, _vp,
                             _i64, _vp, _vp, _vp]),
    "zeus_pso_sweep": (_int, [_int, _int, _i64, _i64, _u64, _int, _dbl, _dbl, _dbl, _vp, _vp,
                              _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "zeus_minloc_select": (_int, [_int, _int, _vp, _vp, _vp, _vp]),
    "zeus_pso_run": (_int, [_int, _int, _i64, _i64, _u64, _dbl, _dbl, _dbl, _dbl, _dbl, _int,
                            _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "zeus_pso_xchg_bytes": (_sz, [_int, _int]),
    "zeus_pso_xchg_setup": (_int, [_vp, _int, _int, _int, ctypes.POINTER(_vp), _vp]),
    "zeus_pso_xchg_status": (_int, [_vp, _int, _int, ctypes.POINTER(ctypes.c_uint)]),
    "zeus_pso_run_xchg": (_int, [_int, _int, _i64, _i64, _u64, _dbl, _dbl, _dbl, _dbl, _dbl,
                                 _int, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _int,
                                 ctypes.c_ulonglong, _vp]),
    "zeus_bfgs_workspace_bytes": (_sz, [_int, _i64]),
    "zeus_bfgs": (_int, [_int, _int, _i64, _vp, _i64, ctypes.POINTER(BfgsParams), _i64, _vp,
                         _vp, ctypes.POINTER(BfgsOut), _vp, _vp]),
    "zeus_argmin_workspace_bytes": (_sz, [_i64]),
    "zeus_reduce_best": (_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "zeus_armijo": (_int, [_int, _int, _i64, _vp, _vp, _vp, _i64, _vp,
                           ctypes.POINTER(BfgsParams), _vp, _vp, _vp]),
    "zeus_hessian_update": (_int, [_int, _i64, _vp, _vp, _vp, _vp, _vp]),
    "zeus_bench_dfma": (_int, [_int, _int, ctypes.c_longlong, _vp,
                               ctypes.POINTER(_dbl), _vp]),
    "zeus_count_within": (_int, [_int, _i64, _vp, _i64, _vp, _dbl, _vp, _vp]),
    "zeus_pack_results": (_int, [ctypes.POINTER(BfgsOut), _int, _i64, _vp, _vp, _vp, _vp, _vp,
                                 _int, _vp, _vp]),
    "zeus_host_device_ptr": (_int, [_vp, ctypes.POINTER(_vp)]),
    "zeus_user_compile": (_int, [ctypes.c_char_p, _int, ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "zeus_user_compile_log": (ctypes.c_char_p, []),
    "zeus_user_free": (_int, [_vp]),
    "zeus_user_dim": (_int, [_vp]),
    "zeus_user_set_data": (_int, [_vp, _vp, _vp]),
    "zeus_user_value": (_int, [_vp, _i64, _vp, _i64, _vp, _vp]),
    "zeus_user_gradient": (_int, [_vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "zeus_user_armijo": (_int, [_vp, _i64, _vp, _vp, _vp, _i64, _vp, ctypes.POINTER(BfgsParams),
                                _vp, _vp, _vp]),
    "zeus_user_pso_init": (_int, [_vp, _i64, _i64, _u64, _dbl, _dbl, _vp, _vp, _vp, _vp, _i64,
                                  _vp, _vp, _vp]),
    "zeus_user_pso_sweep": (_int, [_vp, _i64, _i64, _u64, _int, _dbl, _dbl, _dbl, _vp, _vp, _vp,
                                   _vp, _i64, _vp, _vp, _vp, _vp]),
    "zeus_user_pso_run": (_int, [_vp, _i64, _i64, _u64, _dbl, _dbl, _dbl, _dbl, _dbl, _int,
                                 _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _int,
                                 ctypes.c_ulonglong, _vp]),
    "zeus_user_bfgs_workspace_bytes": (_sz, []),
    "zeus_user_bfgs": (_int, [_vp, _i64, _vp, _i64, ctypes.POINTER(BfgsParams), _i64, _vp, _vp,
                              ctypes.POINTER(BfgsOut), _vp, _vp]),
    "zeus_ipc_alloc": (_int, [_sz, ctypes.POINTER(_vp), ctypes.c_char_p]),
    "zeus_ipc_open": (_int, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "zeus_ipc_close": (_int, [_vp, _int]),
    "zeus_enable_peer_access": (_int, [_int, _int]),
    "zeus_stop_block_create": (_int, [ctypes.POINTER(_vp), ctypes.c_char_p]),
    "zeus_stop_block_open": (_int, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "zeus_stop_block_close": (_int, [_vp, _int]),
    "zeus_stop_block_reset": (_int, [_vp, _vp]),
}
EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_LIB: ctypes.CDLL | None = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the CUDA library; raises if it is absent."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ZeusNativeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.zeus_abi_version() != ABI_VERSION:
            raise ZeusNativeError("libzeus_sm100.so ABI version mismatch; rebuild it")
        _LIB = L
    return _LIB


def check(rc: int, what: str = "zeus") -> None:
    if rc != 0:
        msg = lib().zeus_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise ZeusNativeError(f"{what} failed (rc={rc}): {msg}")
