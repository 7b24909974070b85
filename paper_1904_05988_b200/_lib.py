"""Loader for libpswe.so (the sm_100a CUDA library behind include/pswe.h).

There is no CPU fallback: if the library is missing or no CUDA device is present, every
operator raises. ``symbols()`` lists the exported ABI for the load-only CPU tests.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PSWE_LIB_VARIANT=x loads libpswe_x.so from the same directory (A/B builds of tuning macros)
LIB_PATH = os.path.join(_HERE, "libpswe.so" if not os.environ.get("PSWE_LIB_VARIANT")
                        else f"libpswe_{os.environ['PSWE_LIB_VARIANT']}.so")

_i, _d, _vp = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
_pi = ctypes.POINTER(ctypes.c_int)


class Params(ctypes.Structure):
    """pswe_params == ModelParams (swe.hpp:13-19)."""
    _fields_ = [("radius", _d), ("omega", _d), ("gravity", _d), ("phi_bar", _d), ("nu", _d)]


class BlockConfig(ctypes.Structure):
    """pswe_block_config == BlockConfig (pfasst.hpp:14-20)."""
    _fields_ = [("n_time_steps", _i), ("dt", _d), ("n_iter", _i)]


# name -> (restype, argtypes); mirrors include/pswe.h
SIGNATURES = {
    "pswe_last_error": (ctypes.c_char_p, []),
    "pswe_abi_version": (_i, []),
    "pswe_device_alloc": (_i, [ctypes.c_ulonglong, ctypes.POINTER(_vp)]),
    "pswe_device_free": (_i, [_vp]),
    "pswe_memcpy_h2d": (_i, [_vp, _vp, ctypes.c_ulonglong, _vp]),
    "pswe_memcpy_d2h": (_i, [_vp, _vp, ctypes.c_ulonglong, _vp]),
    "pswe_stream_synchronize": (_i, [_vp]),
    "pswe_dealiased_nlon": (_i, [_i]),
    "pswe_gauss_latitudes": (_i, [_i, _vp, _vp]),
    "pswe_quadrature_tables": (_i, [_i, _vp, _vp, _vp, _vp]),
    "pswe_plan_create": (_i, [_i, _i, _i, _i, ctypes.POINTER(_vp)]),
    "pswe_plan_destroy": (_i, [_vp]),
    "pswe_plan_info": (_i, [_vp, _pi, _pi, _pi, _pi]),
    "pswe_plan_latitudes": (_i, [_vp, _vp, _vp]),
    "pswe_plan_reserve": (_i, [_vp, _i]),
    "pswe_synthesise": (_i, [_vp, _vp, _vp, _i, _vp]),
    "pswe_analyse": (_i, [_vp, _vp, _vp, _i, _vp]),
    "pswe_uv_from_vortdiv": (_i, [_vp, _vp, _vp, _d, _vp, _vp, _i, _vp]),
    "pswe_vortdiv_from_uv": (_i, [_vp, _vp, _vp, _d, _vp, _vp, _i, _vp]),
    "pswe_laplacian": (_i, [_i, _vp, _d, _vp, _i, _i, _vp]),
    "pswe_eval_explicit": (_i, [_vp, ctypes.POINTER(Params), _vp, _vp, _i, _vp]),
    "pswe_eval_implicit": (_i, [_i, ctypes.POINTER(Params), _vp, _vp, _i, _vp]),
    "pswe_eval_imex": (_i, [_vp, ctypes.POINTER(Params), _vp, _vp, _vp, _i, _vp]),
    "pswe_solve_implicit": (_i, [_i, ctypes.POINTER(Params), _vp, _d, _vp, _i, _vp]),
    "pswe_level_create": (_i, [_vp, ctypes.POINTER(Params), _i, ctypes.POINTER(_vp)]),
    "pswe_level_destroy": (_i, [_vp]),
    "pswe_level_ptr": (_vp, [_vp, _i, _i]),
    "pswe_level_info": (_i, [_vp, _pi, _pi]),
    "pswe_spread": (_i, [_vp, _vp, _vp]),
    "pswe_refresh_nodes": (_i, [_vp, _i, _i, _vp]),
    "pswe_sweep": (_i, [_vp, _d, _vp, _vp]),
    "pswe_collocation_residual": (_i, [_vp, _d, _vp, _vp]),
    "pswe_sdc_step": (_i, [_vp, _vp, _d, _i, _vp, _vp]),
    "pswe_pair_create": (_i, [_vp, _vp, ctypes.POINTER(_vp)]),
    "pswe_pair_destroy": (_i, [_vp]),
    "pswe_restrict_space": (_i, [_i, _i, _vp, _vp, _i, _vp]),
    "pswe_interpolate_space": (_i, [_i, _i, _vp, _vp, _i, _vp]),
    "pswe_restrict_states": (_i, [_vp, _vp]),
    "pswe_fas_correction": (_i, [_vp, _d, _vp, _vp]),
    "pswe_fas_correction_ml": (_i, [_vp, _d, _vp, _vp, _vp]),
    "pswe_save_coarse": (_i, [_vp, _vp]),
    "pswe_interpolate_increment_add": (_i, [_vp, _vp, _vp]),
    "pswe_interpolate_states": (_i, [_vp, _vp]),
    "pswe_pfasst_create_serial": (_i, [_vp, ctypes.POINTER(BlockConfig), ctypes.POINTER(_vp)]),
    "pswe_pfasst_create_nccl": (_i, [_vp, ctypes.POINTER(BlockConfig), _i, _i, _vp, ctypes.POINTER(_vp)]),
    "pswe_pfasst3_create_serial": (_i, [_vp, _vp, ctypes.POINTER(BlockConfig), ctypes.POINTER(_vp)]),
    "pswe_pfasst3_create_nccl": (_i, [_vp, _vp, ctypes.POINTER(BlockConfig), _i, _i, _vp, ctypes.POINTER(_vp)]),
    "pswe_nccl_unique_id": (_i, [_vp]),
    "pswe_transport_unique_id": (_i, [_i, _vp]),
    "pswe_pfasst_create_dist": (_i, [_vp, _vp, ctypes.POINTER(BlockConfig), _i, _i, _i, _vp, ctypes.POINTER(_vp)]),
    "pswe_pfasst_set_recv_timeout": (_i, [_vp, _d]),
    "pswe_pfasst3_configure": (_i, [_vp, _i, _i]),
    "pswe_pfasst_run_block_steps": (_i, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pswe_pfasst_destroy": (_i, [_vp]),
    "pswe_pfasst_run_block": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "pswe_pfasst_run_blocks": (_i, [_vp, _vp, _i, _vp, _vp, _vp]),
    "pswe_pfasst_messages": (_i, [_vp, _pi, _i]),
    "pswe_pfasst_schedule": (_i, [_i, _i, _i, _pi, _i]),
    "pswe_pfasst_schedule_ml": (_i, [_i, _i, _i, _i, _pi, _i]),
    "pswe_fp64_peak": (_d, [_i, _i]),
    "pswe_eval_imex_timed": (_i, [_vp, ctypes.POINTER(Params), _vp, _vp, _vp, _i, _vp,
                                  ctypes.POINTER(ctypes.c_float)]),
    "pswe_eval_imex_kernel_times": (_i, [_vp, ctypes.POINTER(Params), _vp, _vp, _vp, _i, _vp,
                                  ctypes.POINTER(ctypes.c_float)]),
}

_lib = None


class PsweError(RuntimeError):
    pass


def lib():
    """The loaded library; raises (no fallback) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PsweError(f"libpswe.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def symbols():
    return list(SIGNATURES)


def check(rc: int):
    if rc != 0:
        raise PsweError(lib().pswe_last_error().decode())
