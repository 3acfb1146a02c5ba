O=gpurun_out/r2r; mkdir -p $O
timeout 900 python -m pytest -q -rA tests/test_gpu_bwd.py > $O/pytest_bwd.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_bwd.log; grep -E "128\)" $O/pytest_bwd.log | grep max-abs | head -12
