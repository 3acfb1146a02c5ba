O=gpurun_out/r2i; mkdir -p $O
timeout 900 python -m pytest -q -rA tests/test_gpu_bwd.py > $O/pytest_bwd.log 2>&1; echo pytest rc=$?; tail -3 $O/pytest_bwd.log; grep -E "bwd .*max-abs" $O/pytest_bwd.log | head -60
