#!/bin/bash
# First-contact GPU diagnostics: each case in its own process with a timeout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
run() { timeout 60 python tools/gpu_debug.py "$@" 2>&1 | tail -12; echo "[exit ${PIPESTATUS[0]}] $*"; }
run spatial 4 64 2 32
run temporal 4 64 2 32
run spatial 2 256 1 64
run spatial 8 300 2 64
run temporal 8 64 2 64
run temporal 200 4 2 64
run spatial 5 256 2 128
run temporal 5 64 2 128
run block 4 64 2 32
run block 8 300 2 64
run block 200 4 2 64
