#!/bin/bash
# Bench the exp2-emulation share (TSF_EMU of 16) and check parity under each.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sweep
for e in ${EMUS:-0 4 6 8}; do
  TSF_EMU=$e timeout 120 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/sweep/emu$e.json 2>&1
  python - "$e" <<'EOF'
import json, sys
e = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sweep/emu{e}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"EMU={e}: {d['value']:.4g} tok/s  step {d['ms_per_step']:.4f} ms  spatial {r['launch_ms']:.4f} ms "
          f"{r['achieved']:.0f} TF/s frac {r['frac']:.3f}  temporal {r['stage_ms_per_step']['temporal']:.4f} ms  clocks {d['clocks']}")
except Exception as ex:
    print("EMU", e, "failed", ex, open(f"gpurun_out/sweep/emu{e}.json").read()[-2000:])
EOF
  TSF_EMU=$e timeout 90 python tools/gpu_debug.py block 8 4096 16 64 | tail -3
  TSF_EMU=$e timeout 90 python tools/gpu_debug.py spatial 4 1000 4 64 iid | tail -3
done
