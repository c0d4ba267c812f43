"""ctypes binding of ``liboptimus_b200.so`` (declarations: include/optimus_b200.h).

There is no fallback: if the library is missing or the device is not sm_100,
every entry point raises (``ExtensionMissing`` / ``DeviceError``).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigError, DeviceError, ExtensionMissing

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "liboptimus_b200.so"

OPTIMUS_EINVAL = -1
OPTIMUS_ENOSYS = -2

_vp, _i32, _i64, _f32 = C.c_void_p, C.c_int, C.c_int64, C.c_float

# name -> (restype, argtypes); mirrors include/optimus_b200.h one to one.
SIGNATURES = {
    "optimus_version": (_i32, []),
    "optimus_last_error": (C.c_char_p, []),
    "optimus_device_sm_count": (_i32, []),
    "optimus_set_attn_trace": (None, [_vp]),
    "optimus_kv_append": (
        _i32,
        [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _i64, _vp, _i32, _vp],
    ),
    "optimus_attn_plan_bounds": (_i32, [_i32, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "optimus_attn_plan": (
        _i32,
        [_i32, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _i32, _vp, _vp],
    ),
    "optimus_paged_attn": (
        _i32,
        [
            _vp, _i64, _i32,            # q, q_stride_tok, n_tok_total
            _vp, _vp, _i64,             # k_cache, v_cache, num_pages
            _vp, _vp, _vp, _vp, _vp,    # q_pos, prompt_len, vis_base, vis_off, vis_words
            _vp, _i32,                  # block_tables, max_pages
            _vp, _vp, _i32,             # work, cta_off, grid
            _vp, _i32,                  # groups, n_groups
            _i32, _i32, _i32, _i32, _i32, _f32,  # block_size, Hq, Hkv, head_dim, page_size, sm_scale
            _vp, _i64,                  # out, out_stride_tok
            _vp, _vp, _i32, _vp,        # ws_o, ws_ml, v_dtype, stream
        ],
    ),
    "optimus_paged_attn_append": (
        _i32,
        [
            _vp, _i64, _i32,            # q, q_stride_tok, n_tok_total
            _vp, _vp, _i64,             # k_new, v_new, new_stride_tok
            _vp, _vp, _i64,             # k_cache, v_cache, num_pages
            _vp, _vp, _vp, _vp, _vp,    # q_pos, prompt_len, vis_base, vis_off, vis_words
            _vp, _i32,                  # block_tables, max_pages
            _vp, _vp, _i32,             # work, cta_off, grid
            _vp, _i32,                  # groups, n_groups
            _i32, _i32, _i32, _i32, _i32, _f32,  # block_size, Hq, Hkv, head_dim, page_size, sm_scale
            _vp, _i64,                  # out, out_stride_tok
            _vp, _vp, _i32, _vp, _vp, _vp,  # ws_o, ws_ml, v_dtype, slot_mapping_out, slot_abs, stream
        ],
    ),
    "optimus_unmask_partials": (_i32, [_vp, _i32, _i64, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "optimus_unmask_finalize": (
        _i32,
        [_vp, _i32, _i32, _i32, _vp, _i32, _f32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp],
    ),
    "optimus_unmask_splits": (_i32, [_i32, _i32]),
    "optimus_v_saturated": (_i32, [_vp, _i32, _vp]),
    "optimus_unmask_commit": (
        _i32,
        [_vp, _i32, _i64, _vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _i32, _vp, _f32, _i32, _vp, _vp, _vp, _vp, _vp,
         _vp, _i64, _vp],
    ),
    "optimus_attn_layers": (
        _i32,
        [_i32, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
         _vp, _i32, _vp, _vp, _i32, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _f32, _vp, _i64, _vp,
         _vp, _i32, _i32, _vp, _vp],
    ),
    "optimus_kv_append_slots": (_i32, [_vp, _vp, _i64, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _i64, _i32, _vp]),
    "optimus_device_plan": (_i32, [_i32, _vp, _i32, _vp, _i32, _i32, _vp, _i64, _vp, _i32, _vp, _vp, _vp, _vp,
                                   _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _i32,
                                   _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp]),
    "optimus_device_apply": (_i32, [_i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i32, _vp, _vp,
                                    _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "optimus_admit_record_ints": (_i32, [_i64, _i32, _i32]),
    "optimus_device_admit": (_i32, [_i32, _vp, _vp, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _i32, _vp]),
    "optimus_device_attn_plan": (_i32, [_i32, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _i32,
                                        _vp, _vp]),
    "optimus_lmhead_splits": (_i32, [_i32]),
    "optimus_unmask_merge_splits": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "optimus_lmhead_unmask_partials": (_i32, [_vp, _i64, _i32, _vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "optimus_paged_attn_combine_dev": (_i32, [_vp, _vp, _i32, _vp, _vp, _i32, _i32, _i32, _vp, _i64, _vp]),
    "optimus_kv_append_dev": (_i32, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _i32, _i32, _i32, _vp,
                                     _vp, _i32, _vp]),
    "optimus_unmask_partials_dev": (_i32, [_vp, _i32, _i64, _vp, _i32, _vp, _i32, _i32, _i32, _vp, _vp]),
    "optimus_device_row_src": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp]),
    "optimus_slot_mapping": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp]),
    "optimus_slot_mapping_dev": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _vp]),
    "optimus_kv_append_slots_dev": (_i32, [_vp, _vp, _i64, _vp, _i32, _vp, _i32, _i32, _i32, _vp, _vp, _i32, _vp]),
    "optimus_host_plan": (_i32, [_i32, _vp, _i32, _vp, _i32, _i32, _vp, _i64, _vp, _i32, _vp, _vp, _vp, _vp,
                                 _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp,
                                 _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp]),
    "optimus_host_apply": (_i32, [_i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i32,
                                  _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
}

_LIB = None


def load(path: os.PathLike | None = None):
    """Load (once) and type the C-ABI library; raise ExtensionMissing if absent."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise ExtensionMissing(
            f"{p} is not built; run `python -m paper_2605_24832_b200.build` "
            "(the B200 path has no CPU fallback)"
        )
    try:
        lib = C.CDLL(str(p))
    except OSError as exc:  # pragma: no cover - environment specific
        raise ExtensionMissing(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        if path is not None and not hasattr(lib, name):
            continue  # another build (tools/ab_lib.py): type what it exports
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def last_error() -> str:
    msg = load().optimus_last_error()
    return msg.decode() if msg else ""


def check(status: int, entry: str) -> None:
    """Map a C status code onto the package's error hierarchy."""
    if status == 0:
        return
    detail = last_error()
    if status == OPTIMUS_EINVAL:
        raise ConfigError(f"{entry}: {detail}")
    raise DeviceError(entry, status, detail)


def call(name: str, *args) -> int:
    return getattr(load(), name)(*args)
