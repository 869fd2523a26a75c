"""ctypes binding of ``libfc2t2_b200.so`` (the C ABI in include/fc2t2_b200.h).

There is no fallback: if the library is missing this module raises on first
use, and every non-zero status code is turned into the reference exception
class it stands for (DomainError, StageError, OrderError, ...).
"""

from __future__ import annotations

import ctypes as ct
import os
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libfc2t2_b200.so"
# A/B experiments may point at an alternative build of the same library
# (e.g. scripts building with different -D flags); the product uses LIB_PATH.
if os.environ.get("FC2T2_LIB_OVERRIDE"):
    LIB_PATH = Path(os.environ["FC2T2_LIB_OVERRIDE"])

OK, EDOMAIN, ESTAGE, EORDER, ECUDA, EWORKSPACE, EVALUE = range(7)
FLAG_DOMAIN = 1
TABLE_FAR, TABLE_NEAR, TABLE_FARNEAR = 0, 1, 2
L2P_VALUE, L2P_GRAD, L2P_HESS, L2P_WGRAD = 1, 2, 4, 8

_vp = ct.c_void_p
_i32, _i64, _sz = ct.c_int, ct.c_int64, ct.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "fc2t2_version": (_i32, []),
    "fc2t2_last_error": (ct.c_char_p, []),
    "fc2t2_launch_count": (_i64, []),
    "fc2t2_profile_enable": (_i32, [_i32]),
    "fc2t2_profile_read": (_i32, [_i32, _vp, _vp, _vp]),
    "fc2t2_profile_timeline": (_i32, [_i32, _vp, _vp, _vp]),
    "fc2t2_engine_create": (_i32, [_i32, _i32, ct.POINTER(_vp)]),
    "fc2t2_engine_destroy": (None, [_vp]),
    "fc2t2_engine_set_table": (_i32, [_vp, _i32, _i32, _i64, _vp, _vp, _vp]),
    "fc2t2_engine_upload": (_i32, [_vp, _vp]),
    "fc2t2_fit_tables": (_i32, [_i32, _i32, _vp, _vp, _vp, ct.c_double, ct.c_double, _vp, _i64,
                                _vp, _vp, _vp]),
    "fc2t2_fit_tables_smem": (_sz, [_i32]),
    "fc2t2_unpack_rows": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp, _vp]),
    "fc2t2_domain_check": (_i32, [_vp, _i64, _vp, _vp]),
    "fc2t2_engine_list_entries": (_i64, [_vp, _i32, _i32]),
    "fc2t2_engine_get_list": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "fc2t2_find_box": (_i32, [_i32, _vp, _i64, _vp, _vp, _vp]),
    "fc2t2_cell_sort_workspace_size": (_sz, [_i32, _i64]),
    "fc2t2_cell_sort": (_i32, [_i32, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "fc2t2_loss_workspace_size": (_sz, [_i64, _i32]),
    "fc2t2_loss": (_i32, [_vp, _vp, _vp, _i64, _i32, ct.c_float, _i32, _vp, _vp, _vp, _sz, _vp]),
    "fc2t2_nonfinite": (_i32, [_vp, _i64, _vp, _vp]),
    "fc2t2_opt_step": (_i32, [_vp, _vp, _vp, _vp, _i64, _i32, ct.c_float, _i64, ct.c_float,
                              _i32, _vp, _vp]),
    "fc2t2_p2m": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fc2t2_p2m_points_workspace_size": (_sz, [_vp, _i32, _i64]),
    "fc2t2_p2m_points": (_i32, [_vp, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "fc2t2_p2m_points_phase": (_i32, [_vp, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _i32, _vp]),
    "fc2t2_m2m": (_i32, [_vp, _i32, _i32, _vp, _vp, _vp]),
    "fc2t2_l2l": (_i32, [_vp, _i32, _i32, _vp, _vp, _i32, _vp]),
    "fc2t2_m2l_issued_flops": (ct.c_double, [_vp, _i32, _i32, _i32]),
    "fc2t2_m2l_workspace_size": (_sz, [_vp, _i32, _i32, _i32]),
    "fc2t2_m2l": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp, _i32, _vp, _sz, _vp]),
    "fc2t2_engine_set_separable": (_i32, [_vp, _vp, _vp, _vp]),
    "fc2t2_engine_separable": (_i32, [_vp]),
    "fc2t2_engine_set_separable_far": (_i32, [_vp, _i32, _vp, _vp, _vp]),
    "fc2t2_engine_set_sep_fusion": (_i32, [_vp, _i32]),
    "fc2t2_expand_workspace_size": (_sz, [_vp, _i32]),
    "fc2t2_weighted_grad": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "fc2t2_expand": (_i32, [_vp, _i32, _vp, _vp, _vp, _sz, _vp]),
    "fc2t2_expand_slab": (_i32, [_vp, _i32, _vp, _vp, _i32, _i32, _vp, _sz, _vp]),
    "fc2t2_expand_up": (_i32, [_vp, _i32, _vp, _i32, _i32, _vp, _sz, _vp]),
    "fc2t2_expand_down": (_i32, [_vp, _i32, _vp, _vp, _i32, _i32, _vp, _sz, _vp]),
    "fc2t2_expand_lowest": (_i32, [_vp]),
    "fc2t2_expand_grid_offset": (_i64, [_vp, _i32, _i32]),
    "fc2t2_expand_slab_split": (_i32, [_vp, _i32, _i32]),
    "fc2t2_l2p": (_i32, [_i32, _i32, _i32, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp,
                         _vp, _vp]),
    "fc2t2_ray_last_error": (ct.c_char_p, []),
    "fc2t2_scan_workspace_size": (_sz, [_i64]),
    "fc2t2_scan_u32": (_i32, [_vp, _vp, _i64, _vp, _sz, _vp]),
    "fc2t2_traverse_count": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp]),
    "fc2t2_traverse_fill": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fc2t2_depth_forward": (_i32, [_i32, _i32, _vp, _vp, _vp, _i64, ct.c_double, _vp, _vp, _vp,
                                   _vp, _vp, _vp, _vp]),
    "fc2t2_root_payload": (_i32, [_i32, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _vp, _vp]),
    "fc2t2_line_integral": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp]),
    "fc2t2_line_payload": (_i32, [_i32, _i32, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i32,
                                  _vp, _vp, _vp]),
    "fc2t2_key_sort_workspace_size": (_sz, [_i32, _i64]),
    "fc2t2_key_sort": (_i32, [_i32, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "fc2t2_insert": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "fc2t2_vol_record_floats": (_i32, [_i32]),
    "fc2t2_vol_insert": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "fc2t2_vol_gauss_nodes": (_i32, [_i32]),
    "fc2t2_vol_forward": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _vp]),
    "fc2t2_vol_forward_ex": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _vp]),
    "fc2t2_vol_totals": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "fc2t2_vol_payload": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _vp, _vp, _vp, _vp, _vp]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def exported_symbols() -> list[str]:
    return list(_SIGS)


def lib():
    """Load the shared library once (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise LibraryMissing(
                f"{LIB_PATH} not found: build it with `python -m paper_2111_00110_b200.build` "
                "(the FC2T2 B200 path has no CPU fallback)")
        handle = ct.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def _exc_for(code: int):
    from .expansion import DomainError, StageError
    from .multiindex import OrderError
    return {EDOMAIN: DomainError, ESTAGE: StageError, EORDER: OrderError,
            EVALUE: ValueError, EWORKSPACE: MemoryError}.get(code, RuntimeError)


def check(code: int, what: str = "") -> None:
    if code != OK:
        msg = lib().fc2t2_last_error().decode(errors="replace")
        rmsg = lib().fc2t2_ray_last_error().decode(errors="replace")
        msg = rmsg if rmsg and not msg else (msg + ("; " + rmsg if rmsg else ""))
        raise _exc_for(code)(f"{what}: {msg}" if what else msg)


def profile_timeline(max_entries: int = 512) -> list:
    """[(kernel name, begin ms, end ms)] of the launches recorded since
    profile_enable(True), in issue order, relative to the first one."""
    import numpy as np
    names = ct.create_string_buffer(32 * max_entries)
    t0 = np.zeros(max_entries, dtype=np.float64)
    t1 = np.zeros(max_entries, dtype=np.float64)
    n = lib().fc2t2_profile_timeline(max_entries, names, t0.ctypes.data, t1.ctypes.data)
    if n < 0:
        check(ECUDA, "profile_timeline")
    raw = names.raw
    return [(raw[32 * k:32 * (k + 1)].split(b"\0", 1)[0].decode(), float(t0[k]), float(t1[k]))
            for k in range(n)]


def launch_count() -> int:
    return int(lib().fc2t2_launch_count())


def profile_enable(on: bool) -> None:
    lib().fc2t2_profile_enable(1 if on else 0)


def profile_read(max_entries: int = 64) -> dict:
    """{kernel name: (total ms, launches)} of the events recorded since
    profile_enable(True); synchronises on those events."""
    import numpy as np
    names = ct.create_string_buffer(32 * max_entries)
    ms = np.zeros(max_entries, dtype=np.float64)
    cnt = np.zeros(max_entries, dtype=np.int64)
    n = lib().fc2t2_profile_read(max_entries, names, ms.ctypes.data, cnt.ctypes.data)
    if n < 0:
        check(ECUDA, "profile_read")
    raw = names.raw
    out = {}
    for k in range(n):
        nm = raw[32 * k:32 * (k + 1)].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[k]), int(cnt[k]))
    return out


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
