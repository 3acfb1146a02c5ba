"""Per-step timeline of CTA 0 of the flash3 kernel (diagnostics).

    python -m paper_2604_16590_b200.build --trace
    TSF_FLASH3=1 TSF_LIB=paper_2604_16590_b200/libtsf_trace.so python tools/trace_flash3.py

Softmax warp w, step j (last item): 0 S ready, 1 max done, 2 P handed.  MMA
warp 5: 0 P seen, 1 PV + next QK^T issued.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import synth
import paper_2604_16590_b200 as tsf


def main():
    K, N, H, d = 8, 4096, 16, 64
    layer = tsf.Layer(K, N, H, d)
    x = synth.bits_to_torch(synth.make_iid(K, N, H, d, seed=0), "cuda")
    for _ in range(3):
        layer.block(x)
    torch.cuda.synchronize()
    L = tsf.lib()
    buf = (ctypes.c_ulonglong * (32 * 1024))()
    L.tsf_trace_read.restype = ctypes.c_int
    L.tsf_trace_read(layer._h, buf, 32 * 1024)
    layer.block(x)
    torch.cuda.synchronize()
    L.tsf_trace_read(layer._h, buf, 32 * 1024)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(32, 1024).astype(np.int64)
    nsub = N // 64
    sm = a[0, :4 * nsub].reshape(nsub, 4)[:, :3]
    mm = a[5, :2 * nsub].reshape(nsub, 2)
    step = np.diff(sm[:, 0])
    print(f"steps {nsub}: cycles/step mean {step.mean():.0f}  (S ready -> max {np.mean(sm[:, 1] - sm[:, 0]):.0f}, "
          f"max -> P handed {np.mean(sm[:, 2] - sm[:, 1]):.0f}, P handed -> MMA sees it {np.mean(mm[:, 0] - sm[:, 2]):.0f}, "
          f"MMA sees P -> issued {np.mean(mm[:, 1] - mm[:, 0]):.0f}, issued -> next S ready "
          f"{np.mean(sm[1:, 0] - mm[:-1, 1]):.0f})")
    t0 = sm[0, 0]
    for j in range(4):
        print(j, (sm[j] - t0).tolist(), (mm[j] - t0).tolist())


if __name__ == "__main__":
    main()
