#!/bin/bash
# Multi-GPU session: build, multi-rank parity tests, bench at 1..N GPUs.  usage: scale_session.sh TAG N
TAG=${1:-r1s}; N=${2:-4}
mkdir -p gpurun_out
python -c "from paper_2603_05800_b200 import build; build.build(); from oracle import oracle; oracle.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/${TAG}_mpytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_mpytest.log
python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench1.json 2> gpurun_out/${TAG}_bench1.err
for g in 2 4 8; do
  [ $g -le $N ] || continue
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2955$g bench.py --gpus $g > gpurun_out/${TAG}_bench$g.json 2> gpurun_out/${TAG}_bench$g.err
done
echo done
