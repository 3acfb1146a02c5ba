#!/bin/bash
# One GPU call: plain bench (the number), then the ncu launch list and one
# `--set full` capture per attention kernel (numbers under ncu are never bench values).
# Usage: bash tools/profile_round.sh <tag>
set -u
cd "$(dirname "$0")/.."
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/smi.txt"
python bench.py --steps 2000 --warmup 10 > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench rc=$?"; cat "$OUT/bench.json"
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline"
$CMD > "$OUT/plain.log" 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_launch.log" 2>&1
echo "launch list rc=$?"
$CMD > "$OUT/plain2.log" 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_ -s 4 -c 2 -o "$OUT/prof" $CMD > "$OUT/ncu_full.log" 2>&1
echo "full capture rc=$?"
ls -la "$OUT"
