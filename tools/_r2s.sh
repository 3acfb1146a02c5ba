O=gpurun_out/r2s; mkdir -p $O
timeout 900 python -m pytest -q -rA tests/test_gpu_dist_sim.py tests/test_gpu_bwd.py -k "bwd or reshard" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest.log
