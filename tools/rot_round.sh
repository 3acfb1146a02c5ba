#!/bin/bash
cd "$(dirname "$0")/.."
timeout 90 python tools/gpu_debug.py block 8 1000 4 64 2>&1 | tail -2
timeout 90 python tools/gpu_debug.py block 1024 64 2 64 2>&1 | tail -2
VARIANTS="96,1,4,0 96,1,6,0 96,1,2,0" bash tools/variant_sweep.sh
NOSWEEP=1 TRACE_FLAGS=0 bash tools/flags_round.sh 2>&1 | tail -16
