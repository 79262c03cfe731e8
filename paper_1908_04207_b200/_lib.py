"""ctypes binding of the C ABI in include/eagercoll_b200.h.

The product path has no fallback: if libeagercoll_b200.so is missing or fails to
load, importing the collective API raises.  (The library is built in-tree by
`python -m paper_1908_04207_b200.build` / `__graft_entry__.build()`.)
"""

from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# EC_DEBUG_LIB=1: the checked build (device assertions, build.py --debug)
LIB_PATH = os.path.join(HERE, "lib", "libeagercoll_b200_debug.so" if os.environ.get("EC_DEBUG_LIB")
                        else "libeagercoll_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "eagercoll_b200.h")

EC_F32, EC_F64, EC_I64 = 0, 1, 2
EC_SYNC, EC_SOLO, EC_MAJORITY = 0, 1, 2
EC_FOLD_COPY, EC_FOLD_ADD = 0, 1
EC_CF_FRESH, EC_CF_ACTIVATE, EC_CF_ALL_ARRIVE = 1, 2, 4
R_PENDING, R_ACCEPTED, R_REFUSED, R_OK, R_POISONED, R_ERROR = 0, 1, 2, 3, 4, 5
E_TIMEOUT = -3
E_DEVICE = -6
INT64_MAX = (1 << 63) - 1
UINT64_MAX = (1 << 64) - 1

_vp = C.c_void_p
_i32, _i64, _u32, _u64 = C.c_int, C.c_int64, C.c_uint32, C.c_uint64
_P = C.POINTER

_SIGS = {
    "ec_version": (_i32, []),
    "ec_last_error": (C.c_char_p, []),
    "ec_launch_count": (_u64, []),
    "ec_comm_create": (_i32, [_i32, _i32, _i32, _i32, _i64, _i32, _i32, _i32, _i32, _P(_vp)]),
    "ec_comm_export": (_i32, [_vp, _i32, _vp, C.c_size_t, _P(C.c_size_t)]),
    "ec_comm_import": (_i32, [_vp, _i32, _vp, C.c_size_t]),
    "ec_comm_set_replay": (_i32, [_vp, _i32, _P(_u64), _i64]),
    "ec_comm_set_quorum": (_i32, [_vp, _i32]),
    "ec_comm_start": (_i32, [_vp]),
    "ec_nvls_supported": (_i32, [_i32]),
    "ec_nvls_create": (_i32, [_vp, _vp, C.c_size_t, _P(C.c_size_t)]),
    "ec_nvls_attach": (_i32, [_vp, _vp, C.c_size_t]),
    "ec_nvls_bind": (_i32, [_vp]),
    "ec_comm_pause": (_i32, [_vp, _i32]),
    "ec_comm_idle_stats": (_i32, [_vp, _P(_u64), _P(_u64), _P(_i32)]),
    "ec_comm_traffic": (_i32, [_vp, _i32, _P(_u64), _P(_u64)]),
    "ec_step_times": (_i32, [_vp, _i32, _i64, _P(_u64)]),
    "ec_step_iterations": (_i32, [_vp, _i32, _i64, _P(_u64)]),
    "ec_comm_destroy": (_i32, [_vp]),
    "ec_comm_error": (_i32, [_vp, _i32, _P(_u64), _P(_u64)]),
    "ec_debug_state": (_i32, [_vp, _i32, _P(_i64)]),
    "ec_send_ptr": (_vp, [_vp, _i32]),
    "ec_grad_ptr": (_vp, [_vp, _i32]),
    "ec_slot_ptr": (_vp, [_vp, _i32, _i64]),
    "ec_n_elems": (_i64, [_vp]),
    "ec_comm_progressive": (_i32, [_vp]),
    "ec_stream_barrier": (_i32, [_vp, _i32, _vp]),
    "ec_comm_set_generation": (_i32, [_vp, _i32, _i64, _i32, _i64]),
    "ec_fold": (_i32, [_vp, _i32, _vp, _i32, _vp]),
    "ec_copy_in": (_i32, [_vp, _i32, _vp, _vp]),
    "ec_post_contribute": (_i32, [_vp, _i32, _i64, _u32, _vp, _P(_u64)]),
    "ec_post_activate": (_i32, [_vp, _i32, _i64, _P(_u64)]),
    "ec_post_hold": (_i32, [_vp, _i32, _i64, _P(_u64)]),
    "ec_post_guard": (_i32, [_vp, _i32, _i64, _i64, _P(_u64)]),
    "ec_reply": (_i32, [_vp, _i32, _u64, _i32, _P(_i32)]),
    "ec_done_gen": (_i32, [_vp, _i32, _P(_i64)]),
    "ec_wait": (_i32, [_vp, _i32, _i64, _i32, _i32, _P(_i64), _P(_u64), _P(_i32)]),
    "ec_gen_info": (_i32, [_vp, _i32, _i64, _P(_u64), _P(_u64), _P(_i32)]),
    "ec_set_pin": (_i32, [_vp, _i32, _u64, _i32, _vp]),
    "ec_gen_times": (_i32, [_vp, _i32, _i64, _P(_u64)]),
    "ec_step_async": (_i32, [_vp, _i32, _i64, _vp, _u32, _vp, _vp, C.c_double, C.c_double, _vp,
                             _P(_u64)]),
    "ec_step_result": (_i32, [_vp, _i32, _u64, _i64, _i32, _P(_i32), _P(_i64), _P(_u64), _P(_i32)]),
    "ec_profile_enable": (_i32, [_i32]),
    "ec_step_update_ns": (_i32, [_vp, _i32, _P(_u64)]),
    "ec_profile_read": (_i32, [_P(C.c_double), _P(_i64)]),
    "ec_round_async": (_i32, [_vp, _i32, _i64, _u32, _vp, _P(_u64)]),
    "ec_round": (_i32, [_vp, _i32, _i64, _u32, _vp, _i32, _P(_i32), _P(_i64), _P(_u64), _P(_i32)]),
    "ec_step": (_i32, [_vp, _i32, _i64, _vp, _i32, _u32, _vp, _vp, C.c_double, C.c_double, _vp,
                       _i32, _P(_i32), _P(_i64), _P(_u64), _P(_i32)]),
    "ec_fold_raw": (_i32, [_vp, _vp, _i64, _i32, _i32, _P(_u32), _vp]),
    "ec_sgd_update": (_i32, [_vp, _vp, C.c_double, _i64, _i32, _vp]),
    "ec_momentum_update": (_i32, [_vp, _vp, _vp, C.c_double, C.c_double, _i64, _i32, _vp]),
    "ec_local_reduce": (_i32, [_P(_vp), _i32, _u64, _vp, _i64, _i32, _i32, _vp]),
    "ec_spin": (_i32, [_u64, _vp]),
}


class EcError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


class EcTimeout(EcError, TimeoutError):
    pass


def header_symbols() -> list[str]:
    """Every function the public header declares (the ABI contract)."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|uint64_t|void\*|const char\*)\s+(ec_\w+)\s*\(",
                                 text, flags=re.M)))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1908_04207_b200.build` "
            "(there is no CPU fallback for this path)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int, fn: str = "ec call") -> int:
    if rc < 0:
        msg = lib.ec_last_error().decode(errors="replace")
        if rc == E_TIMEOUT:
            raise EcTimeout(fn, rc, msg)
        raise EcError(fn, rc, msg)
    return rc


def call(name: str, *args) -> int:
    return check(getattr(lib, name)(*args), name)
