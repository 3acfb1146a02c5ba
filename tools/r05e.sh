cd $GRAFT_REPO_ROOT
O=gpurun_out/r05e; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "temporal_and_spatial or peaky or block_matches or full_C2 or deterministic or degenerate or full_size" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for sp in 2 1; do for fl in 0 2; do for emu in 4 6; do
 TSF_SPLIT=$sp TSF_FLASH_FLAGS=$fl TSF_EMU=$emu timeout 120 python bench.py --steps 600 --warmup 10 --no-cpu-baseline > $O/b_${sp}_${fl}_${emu}.json 2>&1
 python -c "
import json;d=json.loads(open('$O/b_${sp}_${fl}_${emu}.json').read().strip().splitlines()[-1]);r=d['roofline'];print('split $sp flags $fl emu $emu',round(d['value']/1e6,2),'M tok/s', round(r['achieved']),'TF/s frac',round(r['frac'],3), d['clocks']['sm_mhz'])" || tail -3 $O/b_${sp}_${fl}_${emu}.json
done; done; done
TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py > $O/trace_s2.txt 2>&1; head -24 $O/trace_s2.txt
TSF_FLASH_FLAGS=2 TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py > $O/trace_s2pp.txt 2>&1; head -24 $O/trace_s2pp.txt
