"""Timeline of CTA 0 of the streaming temporal kernel (attn_stream.cuh), diagnostics.

    python -m paper_2604_16590_b200.build --trace
    TSF_LIB=paper_2604_16590_b200/libtsf_trace.so python tools/trace_stream.py [K N H d]

Stamps (clock64, CTA 0, trace row 12 + warp): producer warp 16: stage free
(per tile); converter warps 12-15: tile landed / converted; QK warp 17 and PV
warp 18: operands ready; softmax warp 0: S ready / P computed / slot free /
P handed over; epilogue warps 4 / 8 (even / odd tiles): O ready / O read /
staging written / store issued.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import synth
import paper_2604_16590_b200 as tsf

PER_WARP = 1024


def main():
    K, N, H, d = (int(a) for a in sys.argv[1:5]) if len(sys.argv) >= 5 else (8, 4096, 16, 64)
    layer = tsf.Layer(K, N, H, d)
    x = synth.bits_to_torch(synth.make_iid(K, N, H, d, seed=0), "cuda")
    for _ in range(3):
        layer.block(x)
    torch.cuda.synchronize()
    L = tsf.lib()
    n = 32 * PER_WARP
    buf = (ctypes.c_ulonglong * n)()
    L.tsf_trace_read.restype = ctypes.c_int
    L.tsf_trace_read(layer._h, buf, n)
    layer.block(x)
    torch.cuda.synchronize()
    L.tsf_trace_read(layer._h, buf, n)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(32, PER_WARP).astype(np.int64)
    R = 12                                              # the kernel stamps warp w into row 12 + w
    nt = int(np.count_nonzero(a[R + 17]))
    t0 = a[R:][a[R:] > 0].min()
    r = lambda v: (v - t0).tolist()
    print(f"tiles in CTA0: {nt}")
    print("producer stage-free  :", r(a[R + 16, :nt]))
    conv = [a[R + 12 + (i % 4), 2 * (i // 4):2 * (i // 4) + 2] for i in range(nt)]
    print("converter landed     :", r(np.array([c[0] for c in conv])))
    print("converter done       :", r(np.array([c[1] for c in conv])))
    print("QK issue             :", r(a[R + 17, :nt]))
    sm = a[R + 0, :4 * nt].reshape(nt, 4)
    print("softmax S ready      :", r(sm[:, 0]))
    print("softmax P computed   :", r(sm[:, 1]))
    print("softmax slot free    :", r(sm[:, 2]))
    print("softmax P handed     :", r(sm[:, 3]))
    print("PV issue             :", r(a[R + 18, :nt]))
    ep = np.array([a[R + 4 + 4 * (i % 2), 4 * (i // 2):4 * (i // 2) + 4] for i in range(nt)])
    print("epilogue O ready     :", r(ep[:, 0]))
    print("epilogue O read      :", r(ep[:, 1]))
    print("epilogue staged      :", r(ep[:, 2]))
    print("epilogue store issued:", r(ep[:, 3]))
    span = ep[-1, 3] - t0
    cv = np.array([c[1] - c[0] for c in conv])
    print(f"span {span} cycles, {span / nt:.0f} per tile; mean softmax {np.mean(sm[:, 3] - sm[:, 0]):.0f}, "
          f"epilogue {np.mean(ep[:, 3] - ep[:, 0]):.0f}, convert {cv.mean():.0f}")


if __name__ == "__main__":
    main()
