#!/bin/bash
# Flash schedule variants (TSF_FLASH_FLAGS) with parity checks and CTA-0 traces.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
[ -z "$NOSWEEP" ] && CHECK=1 bash tools/variant_sweep.sh
for fl in ${TRACE_FLAGS:-2 0}; do
  TSF_FLASH_FLAGS=$fl TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py > gpurun_out/tr_f$fl.txt 2>&1
  echo "== trace flags $fl"; head -14 gpurun_out/tr_f$fl.txt
done
