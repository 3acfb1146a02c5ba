O=gpurun_out/r2w; mkdir -p $O
for fl in 0 16; do TSF_FLASH_FLAGS=$fl timeout 300 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/c5_$fl.json 2>&1; python -c "
import json;d=json.loads(open('$O/c5_$fl.json').read().strip().splitlines()[-1]);r=d['roofline'];print('C5 flags=$fl', round(d['value']/1e6,2),'Mtok/s',r['stage_ms_per_step'])"; done
timeout 300 python -m pytest -q -x tests/test_gpu_stage_shard.py 2>/dev/null; timeout 600 python -m pytest -q tests/test_gpu_dist_sim.py -k "shard_handle" 2>&1 | tail -1
