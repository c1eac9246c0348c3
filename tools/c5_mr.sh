#!/bin/bash
# C5 at N ranks through bench.py (default settings), twice.  usage: c5_mr.sh N
N=${1:-4}
for i in 1 2; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2972$N bench.py --gpus $N --configs C5 --stream-steps 0 --no-cpu-baseline --e2e-steps 1 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['configs']['C5']; print('default', $N, round(d['ms_per_step'],3), round(v['ms_per_step'],2), v['gpu_launches'], all(v['parity'].values()))"
done
