O=gpurun_out/r2x; mkdir -p $O
timeout 300 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/c5.json 2>&1; python -c "
import json;d=json.loads(open('$O/c5.json').read().strip().splitlines()[-1]);r=d['roofline'];print('C5', round(d['value']/1e6,2),'Mtok/s frac',round(r['frac'],4),r['stage_ms_per_step'])"
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_dist_sim.py -k "block_matches or full_size_block or K200 or 300 or nonfinite or large_config" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest.log
