cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r05k}; mkdir -p $O
for fl in 16 32; do TSF_FLASH_FLAGS=$fl timeout 30 python tools/gpu_debug.py block 8 1000 40 64 | tail -1; done
for v in ${VARS:-1_0_4 1_16_4 1_32_4 1_48_4 1_32_6}; do set -- ${v//_/ }
 TSF_SPLIT=$1 TSF_FLASH_FLAGS=$2 TSF_EMU=$3 timeout 60 python bench.py --steps 600 --warmup 10 --no-cpu-baseline > $O/b_$v.json 2>&1
 python -c "
import json;d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]);r=d['roofline'];print('split/flags/emu $v',round(d['value']/1e6,2),'M tok/s', round(r['achieved']),'TF/s frac',round(r['frac'],3), d['clocks']['sm_mhz'])" || tail -3 $O/b_$v.json
done
for fl in 0 32; do TSF_FLASH_FLAGS=$fl TSF_SPLIT=1 TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 60 python tools/trace_flash.py > $O/trace$fl.txt 2>&1; head -16 $O/trace$fl.txt; done
