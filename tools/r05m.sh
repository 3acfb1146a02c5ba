cd $GRAFT_REPO_ROOT
O=gpurun_out/r05m; mkdir -p $O
TSF_SUB=64 timeout 30 python tools/gpu_debug.py block 8 1000 40 64 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "temporal_and_spatial or peaky or block_matches or full_C2 or deterministic or degenerate" > $O/pytest96.log 2>&1; echo "pytest default rc=$?"; tail -3 $O/pytest96.log
TSF_SUB=64 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "temporal_and_spatial or peaky or block_matches or full_C2 or deterministic or degenerate" > $O/pytest64.log 2>&1; echo "pytest SUB=64 rc=$?"; tail -3 $O/pytest64.log
for v in ${VARS:-96_0_4 64_0_4 64_8_4 64_0_6 64_0_8}; do set -- ${v//_/ }
 TSF_SUB=$1 TSF_FLASH_FLAGS=$2 TSF_EMU=$3 timeout 60 python bench.py --steps 600 --warmup 10 --no-cpu-baseline > $O/b_$v.json 2>&1
 python -c "
import json;d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]);r=d['roofline'];print('sub/flags/emu $v',round(d['value']/1e6,2),'M tok/s', round(r['achieved']),'TF/s frac',round(r['frac'],3), d['clocks']['sm_mhz'])" || tail -3 $O/b_$v.json
done
TSF_SUB=64 TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 60 python tools/trace_flash.py > $O/trace.txt 2>&1; head -12 $O/trace.txt
