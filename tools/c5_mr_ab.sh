#!/bin/bash
# A/B of fold sub-pass settings for C5 at N ranks (bench.py --configs C5). usage: c5_mr_ab.sh N
N=${1:-4}
for spec in "256:256" "512:512" "256:256" "512:512"; do
  mp=$(( ${spec%%:*} << 20 )); sp=$(( ${spec##*:} << 20 ))
  SW_MAX_PASS=$mp SW_SUB_PASS=$sp python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2971$N bench.py --gpus $N --configs C5 --stream-steps 0 --no-cpu-baseline --e2e-steps 1 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['configs']['C5']; print('$spec', $N, round(d['ms_per_step'],3), round(v['ms_per_step'],2), v['gpu_launches'], all(v['parity'].values()))"
done
