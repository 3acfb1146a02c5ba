"""HBM roofline of the layout transpose: tsf_transpose
[A, B, H, d] -> [B, A, H, d] (frame-major <-> token-major) at C2 and C3 sizes.

    python tools/bench_layout.py [reps]

Bytes per launch = read + write of the whole tensor (2 * A*B*H*d*2).  Timed
with CUDA events on the launching stream after warm-up; inputs > L2 (C2: 67 MB
in + 67 MB out alternating between two buffer pairs, C3: 1.07 GB).  Prints one
JSON line per config with GB/s and the fraction of MEASURED_PEAKS hbm_gbs.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2604_16590_b200 as tsf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for name, (K, N, H, d) in {"C2": (8, 4096, 16, 64), "C3": (32, 16384, 16, 64)}.items():
        layer = tsf.Layer(K, N, H, d)
        sets = [(torch.randn(K, N, H, d, device="cuda").to(torch.bfloat16),
                 torch.empty(N, K, H, d, device="cuda", dtype=torch.bfloat16)) for _ in range(2)]
        for i in range(5):
            x, y = sets[i % 2]
            layer.transpose(x, y)
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for i in range(reps):
            x, y = sets[i % 2]
            layer.transpose(x, y)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        x, y = sets[0]
        ok = torch.equal(y, x.transpose(0, 1))
        nbytes = 2 * x.numel() * 2
        gbs = nbytes / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": "transpose_rows_kernel (tsf_transpose)", "config": name, "shape": [K, N, H, d],
                          "bytes_per_launch": nbytes, "ms": ms, "achieved_GBs": gbs, "peak_GBs": peak,
                          "frac": gbs / peak, "exact": ok}))
        layer.close()


if __name__ == "__main__":
    main()
