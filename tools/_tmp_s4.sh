#!/bin/bash
O=gpurun_out/s4; mkdir -p $O
TSF_PARITY_LOG=$O/parity.log timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "short_window or host_batch or host_api" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
run() { env $2 timeout 300 python bench.py $3 --warmup 5 --no-cpu-baseline > "$O/$1.json" 2>/dev/null; echo "$1 rc=$?"; }
run c3_tma8 "TSF_SMALLT=1" "--config C3 --steps 30"
run c3_stream "TSF_SMALLT=0" "--config C3 --steps 30"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/s4/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
        print(f, f"{d['value']:.4g}", "temporal", round(r["stage_ms_per_step"]["temporal"]*1000, 2), "us", d["clocks"]["sm_mhz"])
    except Exception as e: print(f, "ERR", e)
PY
timeout 600 ncu --set full --clock-control none -k regex:attn_smallt -c 2 -o $O/smallt python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/smallt.ncu-rep --page raw --csv > $O/smallt_raw.csv 2>/dev/null
ncu -i $O/smallt.ncu-rep --page details --csv > $O/smallt_details.csv 2>/dev/null
rm -f $O/smallt.ncu-rep
