cd $GRAFT_REPO_ROOT
O=gpurun_out/r05l; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for fl in 0 4; do TSF_FLASH_FLAGS=$fl timeout 300 python bench.py --config C5 --steps 30 --warmup 5 --no-cpu-baseline > $O/c5_$fl.json 2>&1; python -c "
import json;d=json.loads(open('$O/c5_$fl.json').read().strip().splitlines()[-1]);r=d['roofline'];print('C5 flags $fl',d['value'],d['ms_per_step'],r['achieved'],r['frac'],r['stage_ms_per_step'])"; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 tools/dist_check.py 1024 1024 8 64 2>&1 | grep -E "DIST|rank" | tail -3
