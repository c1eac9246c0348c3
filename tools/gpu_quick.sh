#!/bin/bash
# One GPU session: smoke, pytest -m gpu, bench lines.  usage: bash tools/gpu_quick.sh TAG [CONFIGS...]
TAG=${1:-s}; shift; CFGS=${@:-C2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 || { echo "smoke failed"; tail -20 gpurun_out/${TAG}_smoke.log; }
timeout ${PYT_TIMEOUT:-1800} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -15 gpurun_out/${TAG}_pytest.log
for c in $CFGS; do
  timeout 600 python bench.py --config $c ${BENCH_ARGS} > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
done
echo done
