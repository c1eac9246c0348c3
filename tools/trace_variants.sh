#!/bin/bash
# SW_TRACE one-step runs of library variants (tools/build_variant.py) on configs.
# usage: CFGS="C2 C3" bash tools/trace_variants.sh base n8 ...   ("base" = the in-tree library)
mkdir -p gpurun_out
for v in "$@"; do
  for c in ${CFGS:-C2 C3}; do
    if [ "$v" = "base" ]; then unset SW_LIB_VARIANT; else export SW_LIB_VARIANT=$v; fi
    echo "== $v $c"; SW_TRACE=1 timeout 300 python tools/one_step.py $c 3 2>&1 | tail -n 2 | head -1
  done
done
