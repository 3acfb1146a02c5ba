O=gpurun_out/r2u; mkdir -p $O
for P in 2 4; do
  for args in "" "1024 1024 8 64"; do
    tag=$(echo "$args" | tr ' ' '_'); [ -z "$tag" ] && tag=C2weak
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29${P}51 tools/dist_check.py $args > $O/dist_${P}_$tag.log 2>&1; echo "dist P=$P $tag rc=$?"; grep -E "DIST|rank 0" $O/dist_${P}_$tag.log | tail -2 | cut -c1-330
  done
done
