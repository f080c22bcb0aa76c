"""K3 micro-benchmark: the five GEMMs of one reddit_gcn partition step (rows =
ROWS, default 200,000) on device buffers through catgnn_debug_gemm_dev, with
the epilogues the step uses; CUDA-event time per launch (median of REPS) and
the HBM floor of each shape (operand + output bytes / MEASURED_PEAKS hbm).
Checks each result against a float64 torch reference (max relative error).

    python scripts/gemm_micro.py [ROWS] [REPS]
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_02300_b200 import gnnpart as gp  # noqa: E402
from paper_2404_02300_b200._lib import check, lib  # noqa: E402

ROWS = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 20
vp, u32 = C.c_void_p, C.c_uint32
lib.catgnn_debug_gemm_dev.restype = C.c_int
lib.catgnn_debug_gemm_dev.argtypes = [vp, u32, u32, u32, vp, u32, C.c_int, vp, u32, C.c_int, vp, u32, u32, C.c_int,
                                      vp, vp, C.c_int, vp, u32, vp, u32, u32]
try:
    HBM = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    HBM = 6650.0
dev = torch.device("cuda")
stream = torch.cuda.Stream()
ctx = gp.Context(0, stream.cuda_stream)
g = torch.Generator(device="cuda").manual_seed(0)


def rnd(r, c, scale=1.0):
    return (torch.randn(r, c, device=dev, generator=g) * scale).contiguous()


def p(t):
    return t.data_ptr() if t is not None else None


R = ROWS
X = rnd(R, 604)                 # layer-0 input (602 padded to 604)
X[:, 602:] = 0
W0 = rnd(256, 604, 0.05); W0[:, 602:] = 0
H0 = torch.relu(rnd(R, 256))    # hidden activation
W1 = rnd(41, 256, 0.05)
dT1 = rnd(R, 48, 0.01); dT1[:, 41:] = 0
dT0 = rnd(R, 256, 0.01)
dinv = torch.rand(R, device=dev, generator=g) + 0.1
bias1 = torch.zeros(48, device=dev)
bits_words = 8
mask = torch.randint(0, 2**31 - 1, (R, bits_words), device=dev, dtype=torch.int32)
bits_out = torch.zeros(R, bits_words, device=dev, dtype=torch.int32)

cases = {
    # name: (M, N, K, A, lda, a_mn, B, ldb, b_mn, out shape, kwargs, reference)
    "fwd L0  M=rows N=256 K=602": (R, 256, 602, X, 604, 0, W0, 604, 0, (R, 256), dict(rowscale=dinv),
                                   lambda: (X.double() @ W0.double().T) * dinv.double()[:, None]),
    "fwd L1  M=rows N=41 K=256": (R, 41, 256, H0, 256, 0, W1, 256, 0, (R, 48), dict(rowscale=dinv, store=48),
                                  lambda: (H0.double() @ W1.double().T) * dinv.double()[:, None]),
    "dW1     M=41 N=256 K=rows": (41, 256, R, dT1, 48, 1, H0, 256, 1, (41, 256), dict(split=0),
                                  lambda: dT1[:, :41].double().T @ H0.double()),
    "dX1     M=rows N=256 K=41": (R, 256, 41, dT1, 48, 0, W1, 256, 1, (R, 256), dict(mask=True),
                                  None),
    "dW0     M=256 N=602 K=rows": (256, 602, R, dT0, 256, 1, X, 604, 1, (256, 604), dict(split=0),
                                   lambda: dT0.double().T @ X[:, :602].double()),
}
out = {}
for name, (M, N, K, A, lda, amn, B, ldb, bmn, oshape, kw, refn) in cases.items():
    Cm = torch.zeros(*oshape, device=dev)
    mk = mask if kw.get("mask") else None

    def run():
        check(lib.catgnn_debug_gemm_dev(ctx.handle, M, N, K, p(A), lda, amn, p(B), ldb, bmn, p(Cm), oshape[1],
                                        0 if kw.get("split") == 0 else 1, 3, p(kw.get("rowscale")), None, 0,
                                        p(mk), bits_words if mk is not None else 0, None, 0, kw.get("store", 0)))
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(REPS):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream); run(); e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    a_bytes = (K * lda if amn else M * lda) * 4
    b_bytes = (K * ldb if bmn else N * ldb) * 4
    c_bytes = oshape[0] * oshape[1] * 4
    floor = (a_bytes + b_bytes + c_bytes) / (HBM * 1e3)
    err = None
    if refn is not None:
        ref = refn()
        got = Cm[:, :ref.shape[1]].double() if Cm.shape[1] != ref.shape[1] else Cm.double()
        err = float((got - ref).norm() / ref.norm())
    out[name] = dict(us=round(us, 1), floor_us=round(floor, 1), frac_of_floor=round(floor / us, 2),
                     tflops=round(2 * M * N * K / us / 1e6, 1), rel_err=err)
    print(f"{name:30s} {us:8.1f} us  floor {floor:6.1f} us  ({floor / us:4.2f})  "
          f"{2 * M * N * K / us / 1e6:6.1f} TFLOP/s  err {err}", flush=True)
# bf16x3 (precision 4 through catgnn_debug_gemm_dev: operands split on the
# device into hi/lo pairs first — the split is timed separately and excluded)
lib.catgnn_debug_gemm16_dev.restype = C.c_int
lib.catgnn_debug_gemm16_dev.argtypes = [vp, u32, u32, u32, vp, vp, u32, C.c_int, vp, vp, u32, C.c_int, vp, u32, u32,
                                        vp, vp, C.c_int, vp, u32, u32]


def split(t):
    rows, cols = t.shape
    ld8 = (cols + 7) // 8 * 8
    hi = torch.zeros(rows, ld8, device=dev, dtype=torch.bfloat16)
    hi[:, :cols] = t.to(torch.bfloat16)
    lo = torch.zeros(rows, ld8, device=dev, dtype=torch.bfloat16)
    lo[:, :cols] = (t - hi[:, :cols].float()).to(torch.bfloat16)
    return hi, lo, ld8


for name, (M, N, K, A, lda, amn, B, ldb, bmn, oshape, kw, refn) in cases.items():
    Cm = torch.zeros(*oshape, device=dev)
    mk = mask if kw.get("mask") else None
    Ah, Al, la = split(A[:, :(M if amn else K)])
    Bh, Bl, lb = split(B[:, :(N if bmn else K)])

    def run16():
        check(lib.catgnn_debug_gemm16_dev(ctx.handle, M, N, K, p(Ah), p(Al), la, amn, p(Bh), p(Bl), lb, bmn, p(Cm),
                                          oshape[1], 0 if kw.get("split") == 0 else 1, p(kw.get("rowscale")), None,
                                          0, p(mk), bits_words if mk is not None else 0, kw.get("store", 0)))
    run16()
    torch.cuda.synchronize()
    ts = []
    for _ in range(REPS):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream); run16(); e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    err = None
    if refn is not None:
        ref = refn()
        got = Cm[:, :ref.shape[1]].double() if Cm.shape[1] != ref.shape[1] else Cm.double()
        err = float((got - ref).norm() / ref.norm())
    floor = out[name]["floor_us"]
    out[name + " bf16x3"] = dict(us=round(us, 1), floor_us=floor, frac_of_floor=round(floor / us, 2),
                                 tflops=round(2 * M * N * K / us / 1e6, 1), rel_err=err)
    print(f"{name + ' bf16x3':37s} {us:8.1f} us  floor {floor:6.1f} us  ({floor / us:4.2f})  "
          f"{2 * M * N * K / us / 1e6:6.1f} TFLOP/s  err {err}", flush=True)
print(json.dumps({"rows": R, "gemm": out}))
