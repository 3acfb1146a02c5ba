O=gpurun_out/r2p; mkdir -p $O
timeout 1500 python -m pytest -q -x tests -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > $O/bench.json 2>&1; python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);r=d['roofline'];print('C2', round(d['value']/1e6,2),'Mtok/s frac',round(r['frac'],4),r['stage_ms_per_step'],d['clocks']['sm_mhz'])"
timeout 300 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_C5.json 2>&1; python -c "
import json;d=json.loads(open('$O/bench_C5.json').read().strip().splitlines()[-1]);r=d['roofline'];print('C5', round(d['value']/1e6,2),'Mtok/s frac',round(r['frac'],4),r['stage_ms_per_step'],d['clocks']['sm_mhz'])"
for args in "8 4096 16 64" "1024 1024 8 64"; do TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py $args 2>&1 | grep "items in"; done
