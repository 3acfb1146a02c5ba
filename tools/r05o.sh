cd $GRAFT_REPO_ROOT
O=gpurun_out/r05o; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_api or c_abi or block_matches" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > $O/bench.json 2>&1; python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e'], d['gpu_launches'], d['roofline']['achieved'])"
