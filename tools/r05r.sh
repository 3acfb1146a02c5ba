cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/scale
for P in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2958$P \
  tools/dist_check.py 1024 1024 8 64 2>&1 | grep -E "DIST|rank 0|Error|error" | tail -3
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 \
  tools/dist_check.py 200 512 4 64 2>&1 | grep -E "DIST|rank 0|Error|error" | tail -3
for P in 2 4; do P=$P CFGS=C5 TMO=600 bash tools/c5p4.sh 2>&1 | head -1
python -c "
import json;d=json.loads(open('gpurun_out/scale/C5_$P.json').read().strip().splitlines()[-1]);r=d['roofline'];print('C5 P=$P',d['value'],d['ms_per_step'],r['stage_ms_per_step'])"; done
