O=gpurun_out/${TAG:-r2h}; mkdir -p $O
nvidia-smi -L > $O/gpus.txt; NG=$(nvidia-smi -L | wc -l); echo "GPUs: $NG"
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > $O/scale_1.json 2> $O/scale_1.err; echo "P=1 rc=$?"
for P in 2 4; do
  [ $P -gt $NG ] && continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29${P}31 bench.py --gpus $P --steps 500 --warmup 10 > $O/scale_$P.json 2> $O/scale_$P.err; echo "scale P=$P rc=$?"
  for args in "" "200 16 2 64" "128 64 2 128" "1024 1024 8 64"; do
    tag=$(echo "$args" | tr ' ' '_'); [ -z "$tag" ] && tag=C2weak
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29${P}41 tools/dist_check.py $args > $O/dist_${P}_$tag.log 2>&1; echo "dist P=$P $tag rc=$?"; grep -E "DIST|rank" $O/dist_${P}_$tag.log | tail -$((P+1))
  done
done
python - <<'PY'
import json
for P in (1, 2, 4):
    try:
        d = json.loads(open(f"gpurun_out/${TAG:-r2h}/scale_{P}.json").read().strip().splitlines()[-1])
        print(P, round(d["value"] / 1e6, 2), "Mtok/s", round(d["ms_per_step"], 4), "ms/step", d.get("a2a", {}).get("exchange_GBs_per_rank"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(P, "no line", e)
PY
