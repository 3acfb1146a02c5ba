O=gpurun_out/r2e; mkdir -p $O
timeout 900 python -m pytest -q -rA tests/test_gpu_full_block.py tests/test_gpu_storm.py tests/test_gpu_joint.py tests/test_gpu_dist_sim.py tests/test_gpu_parity.py -k "full_block or storm or joint or block_matches or C2_block_every_row and 0 or nonfinite or sim_block or deterministic or temporal_and_spatial" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_stream.py > $O/trace_stream.txt 2>&1; tail -1 $O/trace_stream.txt
for fl in 0 2; do for emu in 4 6 8; do
  echo "== flags=$fl emu=$emu"
  TSF_FLASH_FLAGS=$fl TSF_EMU=$emu timeout 120 python bench.py --steps 600 --warmup 10 --no-cpu-baseline > $O/b_${fl}_$emu.json 2>&1
  python -c "
import json;d=json.loads(open('$O/b_${fl}_$emu.json').read().strip().splitlines()[-1]);r=d['roofline'];print('  value',d['value'],'frac',round(r['frac'],4),'stages',r['stage_ms_per_step'],'clk',d['clocks']['sm_mhz'])"
  TSF_FLASH_FLAGS=$fl TSF_EMU=$emu TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py > $O/trace_${fl}_$emu.txt 2>&1; sed -n 2,3p $O/trace_${fl}_$emu.txt; sed -n 6,6p $O/trace_${fl}_$emu.txt
done; done
TSF_FLASH_FLAGS=2 timeout 300 python tools/gpu_debug.py block 8 1000 40 64 2>&1 | tail -1
TSF_FLASH_FLAGS=2 timeout 300 python tools/gpu_debug.py spatial 8 1000 40 64 iid 2>&1 | tail -1
