"""ctypes binding of the sm_100a library (include/leorzf_b200.h).

The library is loaded lazily on the first kernel call so that the package
imports on CPU-only hosts (tests of the host logic).  There is no CPU
fallback: if the .so is missing or the device is not sm_100, every call
raises NativeLibraryError.
"""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

from .errors import NativeLibraryError

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "_lib" / "libleorzf_b200.so"
HEADER = PKG.parent / "include" / "leorzf_b200.h"

C64, C128 = 0, 1
WS_INVERSE, WS_ARSVD, WS_WOODBURY, WS_CHAIN, WS_PRECODE, WS_RNG = 0, 1, 2, 3, 4, 5

P = C.c_void_p
I32, I64, F64, SZ = C.c_int32, C.c_int64, C.c_double, C.c_size_t


class ArsvdCfg(C.Structure):
    _fields_ = [("eta", C.c_double), ("k_init", C.c_int), ("p", C.c_int),
                ("i_max", C.c_int), ("d_max", C.c_int), ("eta_row", C.c_void_p),
                ("omega_len", C.c_int64)]


class LeoCfg(C.Structure):
    _fields_ = [("K", C.c_int), ("n_x", C.c_int), ("n_y", C.c_int), ("N_RF", C.c_int),
                ("beam_hold", C.c_int), ("nlos_block", C.c_int), ("wavelength", C.c_double),
                ("spacing_m", C.c_double), ("orbit_radius", C.c_double),
                ("orbit_rate", C.c_double), ("pass_s", C.c_double), ("dt", C.c_double),
                ("min_elev_rad", C.c_double), ("atm_loss_dB", C.c_double)]


_SIGS = {
    "lrz_version": (C.c_int, []),
    "lrz_last_error": (C.c_char_p, []),
    "lrz_device_check": (C.c_int, [C.c_int]),
    "lrz_prof_enable": (C.c_int, [C.c_int]),
    "lrz_prof_collect": (C.c_char_p, []),
    "lrz_gram": (C.c_int, [C.c_int, I64, C.c_int, C.c_int, P, I64, F64, P, I64, P]),
    "lrz_gram_delta": (C.c_int, [C.c_int, I64, C.c_int, C.c_int, P, I64, P, I64, C.c_int, P,
                                 I64, P]),
    "lrz_herm_inverse": (C.c_int, [I64, C.c_int, P, I64, P, I64, P, F64, P, P, P]),
    "lrz_arsvd": (C.c_int, [I64, C.c_int, P, I64, P, I64, P, P, C.POINTER(ArsvdCfg), P, P, P,
                            P, P, P, P, P, C.c_int, C.c_int, P, P]),
    "lrz_arsvd_seq": (C.c_int, [I64, C.c_int, C.c_int, P, P, I64, C.POINTER(ArsvdCfg), P, P, P,
                                P, P, P, P, P, P, P, P, C.c_int, P, P]),
    "lrz_arsvd_walk": (C.c_int, [I64, C.c_int, C.c_int, P, P, I64, C.POINTER(ArsvdCfg), P, P, P,
                                 P, P]),
    "lrz_woodbury": (C.c_int, [I64, C.c_int, C.c_int, P, P, I64, P, P, P, P, P, P, P, P, P]),
    "lrz_chain": (C.c_int, [I64, C.c_int, C.c_int, C.c_int, P, P, P, P, P, P, P, P, P, P, P, P,
                            P]),
    "lrz_chain_steps": (C.c_int, [I64, C.c_int, C.c_int, C.c_int, P, P, P, P, P, P, P, P, P, P,
                                  P, P, P]),
    "lrz_precode_rate": (C.c_int, [C.c_int, I64, C.c_int, C.c_int, P, I64, P, I64, F64, P, I64,
                                   P, I64, P, F64, P, P, P, P, P, P, P]),
    "lrz_cgemm": (C.c_int, [C.c_int, I64, C.c_int, C.c_int, C.c_int, C.c_int, P, I64, I64,
                            C.c_int, P, I64, I64, P, I64, I64, P]),
    "lrz_axpby": (C.c_int, [C.c_int, I64, F64, P, F64, P, P, P]),
    "lrz_fro2": (C.c_int, [C.c_int, I64, I64, P, I64, P, P]),
    "lrz_sinr_rate": (C.c_int, [C.c_int, I64, C.c_int, P, I64, P, P, I64, P, P, P, P]),
    "lrz_plan": (C.c_int, [I64, C.c_int, P, P, P, P]),
    "lrz_rng_normals": (C.c_int, [I64, I64, P, P, P, P, P, P, P, P]),
    "lrz_rng_locate": (C.c_int, [I64, I64, P, P, P, P, P, P, P]),
    "lrz_channels": (C.c_int, [C.c_int, I64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P,
                               I64, P, P]),
    "lrz_leo_snapshot": (C.c_int, [C.POINTER(LeoCfg), I64, C.c_int, C.c_int, P, P, P, I64, P,
                                   P, P, P, P, P, P]),
    "lrz_hybrid_precode_rate": (C.c_int, [I64, C.c_int, C.c_int, C.c_int, C.c_int, P, P, P, P,
                                          P, F64, P, I64, P, P, P, P, P, P]),
    "lrz_campaign_reduce": (C.c_int, [I64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P,
                                      P, P]),
    "lrz_workspace_bytes": (SZ, [C.c_int, C.c_int, I64, C.c_int, C.c_int, C.c_int]),
    "lrz_campaign_summary": (C.c_int, [C.c_int, I64, C.c_int, P, P, P, P, P, P]),
    "lrz_update_inverse_ws": (SZ, [C.c_int, I64, C.c_int, C.c_int, C.c_int]),
    "lrz_update_inverse": (C.c_int, [C.c_int, I64, C.c_int, C.c_int, P, P, F64, P, P, P, I64, P,
                                     C.POINTER(ArsvdCfg), P, P, P, P, P, P, P, P, P]),
    "lrz_trajectory_ws": (SZ, [C.c_int, I64, C.c_int, C.c_int, C.c_int, C.c_int]),
    "lrz_trajectory": (C.c_int, [C.c_int, I64, C.c_int, C.c_int, C.c_int, P, F64, F64, P, I64,
                                 C.c_int, C.POINTER(ArsvdCfg), P, I64, P, P, P, P, P, P, P, P,
                                 P, P, P, P, P]),
    "lrz_spec_verify": (C.c_int, [I64, C.c_int, C.c_int, C.POINTER(ArsvdCfg), P, P, P, P, P, P,
                                  P, P, P]),
    "lrz_spec_verify_vote": (C.c_int, [I64, C.c_int, C.c_int, C.POINTER(ArsvdCfg), P, P, P, P, P,
                                       P, P, P, P, P]),
}

_lib = None
_checked_devices: set = set()


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(lrz_\w+)\s*\(", text,
                                 flags=re.M)))


def load() -> C.CDLL:
    """Load the library and declare argument types (no device access)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2512_16543_b200.build` "
            "(there is no CPU fallback)")
    try:
        lib = C.CDLL(str(LIB_PATH))
    except OSError as e:  # pragma: no cover
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib_for(device) -> C.CDLL:
    """The library, after checking that `device` is an sm_100 GPU."""
    lib = load()
    idx = device.index if device.index is not None else 0
    if idx not in _checked_devices:
        if lib.lrz_device_check(idx) != 0:
            raise NativeLibraryError(lib.lrz_last_error().decode())
        _checked_devices.add(idx)
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeLibraryError(f"{what} failed ({rc}): {load().lrz_last_error().decode()}")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(device) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream
