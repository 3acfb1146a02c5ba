cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r05j}; mkdir -p $O
timeout 120 bash tools/r05h.sh
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "temporal_and_spatial or peaky or block_matches or full_C2 or deterministic or degenerate" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for v in ${VARS:-1_0_4 1_0_6 1_8_4 1_2_4 1_2_6}; do set -- ${v//_/ }
 TSF_SPLIT=$1 TSF_FLASH_FLAGS=$2 TSF_EMU=$3 timeout 60 python bench.py --steps 600 --warmup 10 --no-cpu-baseline > $O/b_$v.json 2>&1
 python -c "
import json;d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]);r=d['roofline'];print('split/flags/emu $v',round(d['value']/1e6,2),'M tok/s', round(r['achieved']),'TF/s frac',round(r['frac'],3), d['clocks']['sm_mhz'])" || tail -3 $O/b_$v.json
done
TSF_SPLIT=1 TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 60 python tools/trace_flash.py > $O/trace.txt 2>&1; head -16 $O/trace.txt
