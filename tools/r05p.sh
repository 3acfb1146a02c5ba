cd $GRAFT_REPO_ROOT
O=gpurun_out/r05p; mkdir -p $O
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "temporal_and_spatial or peaky or block_matches or full_C2 or deterministic or degenerate or host_api" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for rep in 1 2; do for fl in 0 16; do
 TSF_FLASH_FLAGS=$fl timeout 60 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > $O/b_${fl}_$rep.json 2>&1
 python -c "
import json;d=json.loads(open('$O/b_${fl}_$rep.json').read().strip().splitlines()[-1]);r=d['roofline'];print('flags $fl rep $rep',round(d['value']/1e6,2),'M tok/s', round(r['achieved']),'TF/s frac',round(r['frac'],3), d['clocks']['sm_mhz'])" || tail -3 $O/b_${fl}_$rep.json
done; done
for fl in 0 16; do TSF_FLASH_FLAGS=$fl timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > $O/c3_$fl.json 2>&1; python -c "
import json;d=json.loads(open('$O/c3_$fl.json').read().strip().splitlines()[-1]);r=d['roofline'];print('C3 flags $fl',d['value'],r['achieved'],r['frac'])"; done
