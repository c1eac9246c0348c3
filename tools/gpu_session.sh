#!/bin/bash
# One GPU session: tests, bench, launch list, ncu --set full of the eval kernel.
# usage: bash tools/gpu_session.sh TAG [CONFIG]
TAG=${1:-r1}; CFG=${2:-C2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python -c "from paper_2603_05800_b200 import build; build.build(); from oracle import oracle; oracle.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 || { echo "smoke failed"; tail -5 gpurun_out/${TAG}_smoke.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --config $CFG > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
[ "${NCU:-1}" = "0" ] && { echo done; exit 0; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --stream-steps 0 > gpurun_out/${TAG}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 3 -c 1 \
   -o gpurun_out/${TAG}_eval python tools/one_step.py $CFG 5 > gpurun_out/${TAG}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s ${SCAN_SKIP:-5} -c 1 \
   -o gpurun_out/${TAG}_scan python tools/one_step.py $CFG 5 > gpurun_out/${TAG}_ncu_scan.log 2>&1
echo done
