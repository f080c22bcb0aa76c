"""ctypes wrapper of upstream/_ref/libspring_ref.so (the reference's SPRING,
used only to prepare bench inputs before any timed region)."""
import ctypes as C
import os

import numpy as np

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libspring_ref.so")


def spring_homes(edge_file: str, num_ids: int, partitions: int, beta=1.05, tau_vol=0, seed=0,
                 add_reverse=False):
    """Per-external-id SPRING home partition (spring.hpp:106-107); returns (home, tau_used)."""
    if not os.path.exists(LIB):
        raise FileNotFoundError(f"{LIB} missing: run `make -C upstream` where /root/reference exists")
    lib = C.CDLL(LIB)
    lib.spring_last_error.restype = C.c_char_p
    home = np.full(num_ids, 0xFFFFFFFF, np.uint32)
    tau = C.c_uint64()
    rc = lib.spring_homes(str(edge_file).encode(), int(add_reverse), C.c_uint32(partitions), C.c_double(beta),
                          C.c_uint64(tau_vol), C.c_uint64(seed), home.ctypes.data_as(C.c_void_p),
                          C.c_uint64(num_ids), C.byref(tau))
    if rc != 0:
        raise RuntimeError(f"SPRING failed [{rc}]: {lib.spring_last_error().decode()}")
    return home, tau.value
