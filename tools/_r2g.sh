O=gpurun_out/r2g; mkdir -p $O
TSF_FLASH3=1 timeout 300 python tools/gpu_debug.py block 8 1000 40 64 2>&1 | tail -1
TSF_FLASH3=1 TSF_F3CTAS=4 timeout 300 python tools/gpu_debug.py block 8 1000 40 64 2>&1 | tail -1
for v in "0 3" "1 3" "1 4"; do set -- $v
  TSF_FLASH3=$1 TSF_F3CTAS=$2 timeout 120 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > $O/b_$1_$2.json 2>&1
  python -c "
import json;d=json.loads(open('$O/b_$1_$2.json').read().strip().splitlines()[-1]);r=d['roofline'];print('flash3=$1 ctas=$2', round(d['value']/1e6,2),'Mtok/s frac',round(r['frac'],4),'stages',r['stage_ms_per_step'],'clk',d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 $O/b_$1_$2.json
done
for c in 3 4; do TSF_FLASH3=1 TSF_F3CTAS=$c TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash3.py 2>&1 | tail -6; done
