O=gpurun_out/r2f; mkdir -p $O
timeout 300 python tools/gpu_debug.py block 8 1000 40 64 2>&1 | tail -1
timeout 300 python tools/gpu_debug.py spatial 8 1000 40 64 iid 2>&1 | tail -1
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_dist_sim.py -k "block_matches or temporal_and_spatial or peaky or C2_block_every_row and 0 or deterministic or sim_block or full_size" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
for v in "0 4" "1 0" "1 2" "1 4" "1 6"; do set -- $v
  TSF_FLASH3=$1 TSF_EMU3=$2 timeout 120 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > $O/b_$1_$2.json 2>&1
  python -c "
import json;d=json.loads(open('$O/b_$1_$2.json').read().strip().splitlines()[-1]);r=d['roofline'];print('flash3=$1 emu3=$2', round(d['value']/1e6,2),'Mtok/s frac',round(r['frac'],4),'stages',r['stage_ms_per_step'],'clk',d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 $O/b_$1_$2.json
done
