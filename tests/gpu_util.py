"""Helpers for the -m gpu tests: device-pointer access to the batched primitives."""
import ctypes as C

import paper_2503_17535_b200 as H

_done = False


def lib():
    global _done
    L = H.lib()
    if not _done:
        vp = C.c_void_p
        L.hpsg_dev_dgemm.argtypes = [C.c_int] * 4 + [C.c_double, vp, C.c_longlong, C.c_longlong, vp, C.c_longlong,
                                                     C.c_longlong, C.c_double, vp, C.c_longlong, C.c_longlong, vp,
                                                     C.c_longlong, C.c_longlong]
        L.hpsg_dev_getrf_aug.argtypes = [C.c_int] * 3 + [vp, C.c_longlong, C.c_longlong, vp, vp]
        L.hpsg_dev_getrs.argtypes = [C.c_int] * 3 + [vp, C.c_longlong, C.c_longlong, vp, vp, C.c_longlong,
                                                     C.c_longlong]
        _done = True
    return L
