#!/bin/bash
# Source-level ncu capture (stall reasons per SASS line) of the spatial flash
# kernel, after a plain run of the same command exits 0.
cd "$(dirname "$0")/.."
OUT=gpurun_out/${1:-src}
mkdir -p "$OUT"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > "$OUT/plain.log" 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_flash -c 1 -o "$OUT/flash" $CMD > "$OUT/ncu.log" 2>&1
echo "ncu rc=$?"; tail -3 "$OUT/ncu.log"
