"""Thin wrappers over the library's launch counter and per-kernel event timers."""
from __future__ import annotations

import ctypes as C

from . import _capi as A


def launch_count() -> int:
    return int(A.lib().spct_cu_launch_count())


def enable(on: bool = True) -> None:
    A.lib().spct_cu_profile_enable(1 if on else 0)


def reset() -> None:
    A.lib().spct_cu_profile_reset()


def kernel_time(name: str) -> tuple[float, int]:
    """(summed device ms, launches) of a bracketed kernel since the last reset."""
    ms, n = C.c_double(), C.c_int()
    A.check(A.lib().spct_cu_profile_read(name.encode(), C.byref(ms), C.byref(n)))
    return ms.value, n.value
