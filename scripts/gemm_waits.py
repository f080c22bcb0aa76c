"""Diagnostics: where the warps of one K3 GEMM shape wait (GEMM_WAIT_PROFILE build,
scripts/build_variant.sh waits "-DGEMM_WAIT_PROFILE"; CATGNN_LIB=<variant>).
Env: SHAPES="M,N,K,a_mn,b_mn;..." (default: the reddit shard-0 GEMMs)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_02300_b200 import gnnpart as gp  # noqa: E402
from paper_2404_02300_b200._lib import lib  # noqa: E402

SITES = ["producer empty", "MMA tempty", "MMA conv", "conv full", "conv lo-slot", "epi tfull"]
shapes = os.environ.get("SHAPES", "184532,41,256,0,0;184532,256,604,0,0;184532,256,41,0,1;41,256,184532,1,1;256,604,184532,1,1")
ctx = gp.Context(0)
lib.catgnn_debug_gemm_waits.argtypes = [C.POINTER(C.c_ulonglong)]
lib.catgnn_gemm.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                            C.c_void_p, C.c_uint32, C.c_int]
out = (C.c_ulonglong * 8)()
for sh in shapes.split(";"):
    M, N, K, amn, bmn = [int(x) for x in sh.split(",")]
    rng = np.random.default_rng(0)
    A = rng.standard_normal((K, M) if amn else (M, K), dtype=np.float32)
    B = rng.standard_normal((K, N) if bmn else (N, K), dtype=np.float32)
    Cm = np.empty((M, N), np.float32)
    args = (ctx.handle, M, N, K, A.ctypes.data, amn, B.ctypes.data, bmn, Cm.ctypes.data, 0, 3)
    lib.catgnn_gemm(*args)
    lib.catgnn_debug_gemm_waits(out)
    lib.catgnn_gemm(*args)
    lib.catgnn_debug_gemm_waits(out)
    print(f"M={M} N={N} K={K} a_mn={amn} b_mn={bmn}: " +
          ", ".join(f"{SITES[i]} {out[i] / 1e3 / 148:.1f} us/CTA" for i in range(6)), flush=True)
