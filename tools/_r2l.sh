O=gpurun_out/r2l; mkdir -p $O
TSF_FLASH_FLAGS=8 timeout 300 python tools/gpu_debug.py block 8 1000 40 64 2>&1 | tail -1
TSF_FLASH_FLAGS=10 timeout 300 python tools/gpu_debug.py block 8 1000 40 64 2>&1 | tail -1
TSF_FLASH_FLAGS=10 timeout 300 python tools/gpu_debug.py spatial 8 1000 40 64 iid 2>&1 | tail -1
for fl in 0 8 10; do for emu in 4 6 8; do
  TSF_FLASH_FLAGS=$fl TSF_EMU=$emu timeout 120 python bench.py --steps 800 --warmup 10 --no-cpu-baseline > $O/b_${fl}_$emu.json 2>&1
  python -c "
import json;d=json.loads(open('$O/b_${fl}_$emu.json').read().strip().splitlines()[-1]);r=d['roofline'];print('flags=$fl emu=$emu', round(d['value']/1e6,2),'Mtok/s frac',round(r['frac'],4),'spatial',round(r['launch_ms'],4),'clk',d['clocks']['sm_mhz'])"
done; done
for fl in 8 10; do TSF_FLASH_FLAGS=$fl TSF_EMU=6 TSF_LIB=paper_2604_16590_b200/libtsf_trace.so timeout 120 python tools/trace_flash.py > $O/trace_$fl.txt 2>&1; sed -n 2,3p $O/trace_$fl.txt; sed -n 6,6p $O/trace_$fl.txt; done
