"""ctypes binding of ``libzstripe_b200.so`` (the C ABI in ``include/zstripe_b200.h``).

This module is the only place Python touches the native library.  It fails
loudly: a missing or stale library raises at import of the first op, and
every non-zero ``zs_status`` becomes a ``RuntimeError`` carrying the
library's own status string.  There is no CPU fallback anywhere.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libzstripe_b200.so"

_p = C.c_void_p
_i = C.c_int
_ll = C.c_longlong
_f = C.c_float
_sz = C.c_size_t

# name -> argtypes (restype is c_int unless noted)
SIGNATURES: dict[str, list] = {
    "zs_abi_version": [],
    "zs_sobel_saliency": [_p, _i, _i, _i, _i, _i, _p, _p, _p],
    "zs_rank_order": [_p, _i, _i, _i, _i, _i, _i, _i, _p, _p, _p, _p],
    "zs_permute_rows_f32": [_p, _p, _p, _ll, _i, _p],
    "zs_permute_rows_bf16": [_p, _p, _p, _ll, _i, _p],
    "zs_permute_rows_f32_bf16": [_p, _p, _p, _ll, _i, _p],
    "zs_layout_maps": [_p, _p, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p],
    "zs_prefix_keep_rows": [_i, _i, _i, _p, _p, _p, _p],
    "zs_unit_span_rows": [_i, _i, _i, _i, _p, _p, _p, _p],
    "zs_layernorm_rows": [_p, _ll, _p, _ll, _i, _p, _p, _f, _p, _ll, _i, _p],
    "zs_layernorm_rows_ex": [_p, _ll, _p, _p, _ll, _p, _i, _p, _p, _f, _p, _ll, _i, _p],
    "zs_gemm_bf16": [_i, _p, _ll, _p, _ll, _i, _i, _i, _p, _p, _ll, _p, _ll, _p, _p, _i, _p, _p],
    "zs_launch_counter": [],  # returns unsigned long long
    "zs_stripe_attn_ws_bytes": [_i, _i, _i, _i, _i, _i],  # returns size_t
    "zs_stripe_attn_fwd": [_p, _p, _p, _ll, _ll, _ll, _ll, _ll, _i, _i, _i, _i, _i, _p, _p, _i, _p, _p, _i, _i,
                           _i, _f, _p, _ll, _ll, _p, _sz, _p],
    "zs_stripe_attn_fwd_rows": [_p, _p, _p, _ll, _ll, _ll, _ll, _ll, _i, _i, _i, _i, _i, _p, _p, _i, _p, _p, _i, _i,
                                _i, _f, _p, _ll, _ll, _p, _p, _sz, _p],
    "zs_stripe_attn_fwd_unit_bias": [_p, _p, _p, _ll, _ll, _ll, _ll, _ll, _i, _i, _i, _i, _i, _p, _p, _ll, _i, _p,
                                     _p, _i, _i, _i, _f, _p, _ll, _ll, _p, _p, _sz, _p],
    "zs_relpos_ws_bytes": [_i, _i, _i, _i, _i],  # returns size_t
    "zs_relpos_bias": [_p, _ll, _ll, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _sz, _p],
    "zs_stripe_attn_fwd_relpos": [_p, _p, _p, _ll, _ll, _ll, _ll, _ll, _i, _i, _i, _i, _p, _p, _i, _p, _p, _i, _i, _i,
                                  _f, _p, _ll, _ll, _p, _p, _sz, _p],
    "zs_invert_rows": [_p, _ll, _p, _p, _ll, _p],
    "zs_fill_flagged_rows_bf16": [_p, _ll, _p, _p, _ll, _i, _p],
    "zs_rc_mlp_fwd": [_p, _ll, _p, _i, _p, _i, _i, _p, _p, _f, _p, _p, _p, _p, _i, _p, _i, _p, _p, _p],
    "zs_patchify": [_p, _i, _i, _i, _i, _i, _p, _p],
    "zs_im2col3x3": [_p, _i, _i, _i, _i, _p, _p],
}

ABI_VERSION = 200
_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load (once) and type the native library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 kernels)"
        )
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_LOCAL", 0))
    lib.zs_status_string.restype = C.c_char_p
    lib.zs_status_string.argtypes = [_i]
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _i
    lib.zs_relpos_ws_bytes.restype = _sz
    lib.zs_stripe_attn_ws_bytes.restype = _sz
    lib.zs_launch_counter.restype = C.c_ulonglong
    if lib.zs_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{LIB_PATH} has ABI {lib.zs_abi_version()}, expected {ABI_VERSION}: rebuild it")
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return ["zs_status_string", *SIGNATURES.keys()]


def status_string(rc: int) -> str:
    return load().zs_status_string(rc).decode()


# kernels launched through the library, counted by the library itself (zs_launch_counter: every
# <<<>>> site in csrc/ increments a per-thread counter), so composites and optional prep kernels
# are counted exactly
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    lib = load()
    n0 = lib.zs_launch_counter()
    rc = getattr(lib, name)(*args)
    launch_count += lib.zs_launch_counter() - n0
    if rc != 0:
        raise RuntimeError(f"{name} failed: zs_status {rc} ({status_string(rc)})")
