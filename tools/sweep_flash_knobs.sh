mkdir -p gpurun_out/sweep
for sub in 96 128 64; do for emu in 4 6 8 0; do
  TSF_SUB=$sub TSF_EMU=$emu timeout 120 python bench.py --no-cpu-baseline --steps 300 --warmup 5 2>/dev/null | python -c "import sys,json; l=json.loads(sys.stdin.read()); print('sub=$sub emu=$emu', round(l['value']/1e6,2), 'Mtok/s frac', round(l['roofline']['frac'],4))" >> gpurun_out/sweep/sweep.txt 2>&1
done; done
cat gpurun_out/sweep/sweep.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/sweep/launches.csv python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/sweep/ncu.log 2>&1; echo ncu_exit=$?
