#!/bin/bash
# Round-2 GPU session: smoke, pytest -m gpu, bench, and ncu captures exported on the box
# (raw metrics + SASS source page as CSV; the .ncu-rep stays on the box).
# usage: TAG=g4 CFG=C2 CONFIGS=C3,C5 NCU="eval:C2 scan:C3" bash tools/gpu_round2.sh
TAG=${TAG:-s}; CFG=${CFG:-C2}; CONFIGS=${CONFIGS:-C2x,C3,C4,C5}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 || { echo "smoke failed"; tail -20 gpurun_out/${TAG}_smoke.log; }
if [ "${PYTEST:-1}" = "1" ]; then
  timeout ${PYT_TIMEOUT:-1800} python -m pytest tests -m gpu -q ${PYTEST_ARGS:---timeout=300 -rf} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -15 gpurun_out/${TAG}_pytest.log
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --config $CFG --configs $CONFIGS ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
fi
cap() {  # name, kernel regex, skip, cmd...
  local n=$1 k=$2 s=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/$n "$@" > gpurun_out/${n}_ncu.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/${n}_raw.csv 2>&1
  ncu -i /tmp/$n.ncu-rep --page source --csv --print-source sass > gpurun_out/${n}_sass.csv 2>&1
  ncu -i /tmp/$n.ncu-rep --page details > gpurun_out/${n}_details.txt 2>&1
}
for t in $NCU; do
  kind=${t%%:*}; c=${t##*:}
  case $kind in
    eval) cap ${TAG}_eval_$c eval_kernel 2 python tools/one_step.py $c 3 ;;
    scan) cap ${TAG}_scan_$c scan_kernel ${SCAN_SKIP:-8} python tools/one_step.py $c 3 ;;
    exact) cap ${TAG}_exact_$c pareto_exact_kernel 5 python tools/one_step.py $c 3 ;;
    eval5) cap ${TAG}_eval_C5 eval_kernel 2 python tools/one_step_c5.py ;;
    scan5) cap ${TAG}_scan_C5 scan_kernel 8 python tools/one_step_c5.py
        SW_DEBUG=1 timeout 300 python tools/one_step_c5.py > gpurun_out/${TAG}_debug_C5chunk.txt 2>&1 ;;
    stream) cap ${TAG}_stream_$c stream_kernel 3 python tools/stream_one.py $c ;;
    launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_$c.csv \
        python bench.py --config $c --configs "" --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --stream-steps 0 > gpurun_out/${TAG}_ncu_launch_$c.log 2>&1
        python tools/launch_summary.py gpurun_out/${TAG}_launches_$c.csv > gpurun_out/${TAG}_launch_summary_$c.txt 2>&1 ;;
    trace) SW_TRACE=1 timeout 300 python tools/one_step.py $c 3 > gpurun_out/${TAG}_trace_$c.txt 2>&1 ;;
    debug) SW_DEBUG=1 SW_TRACE=1 timeout 300 python tools/one_step.py $c 2 > gpurun_out/${TAG}_debug_$c.txt 2>&1 ;;
    dump) mkdir -p gpurun_out/dump; SW_DUMP_MERGE=gpurun_out/dump/${TAG}_$c SW_DEBUG=1 timeout 300 python tools/one_step.py $c 1 > gpurun_out/${TAG}_dump_$c.txt 2>&1 ;;
    sdebug) SW_DEBUG=1 SW_TRACE=1 timeout 300 python tools/shared_one.py $c > gpurun_out/${TAG}_sdebug_$c.txt 2>&1 ;;
  esac
done
du -sh gpurun_out; echo done
