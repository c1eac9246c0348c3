#!/bin/bash
# Bench experiment variants of libsw_plan.so (tools/build_variant.py) on one config.
# usage: CFG=C2 bash tools/gpu_variants.sh base mb5 un2 ...   ("base" = the in-tree library)
CFG=${CFG:-C2}; mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "base" ]; then unset SW_LIB_VARIANT; else export SW_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --config $CFG --configs "${CONFIGS:-}" --stream-steps 0 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/var_${v}_${CFG}.json 2> gpurun_out/var_${v}_${CFG}.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/var_${v}_${CFG}.json'))
k=d['roofline']['kernels']
print('$v', '$CFG', round(d['ms_per_step'],3), 'eval', round(k['eval_kernel']['ms_per_launch'],3), round(k['eval_kernel']['frac'],3), 'scan', round(k['scan_kernel']['ms_per_launch'],3), d['parity'])" 2>&1
done
echo done
