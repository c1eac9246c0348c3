#!/bin/bash
# Stream-mode lines of library variants (tools/build_variant.py) on C2 + configs.
# usage: CONFIGS=C3,C5 bash tools/gpu_stream_variants.sh base smb1
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "base" ]; then unset SW_LIB_VARIANT; else export SW_LIB_VARIANT=$v; fi
  timeout 900 python bench.py --config C2 --configs "${CONFIGS:-C3}" --stream-steps 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/svar_${v}.json 2> gpurun_out/svar_${v}.err
  python -c "
import json; d=json.load(open('gpurun_out/svar_${v}.json'))
out=['$v', 'C2', round(d['ms_per_step'],3), round(d['stream_mode']['ms_per_call'],3), d['stream_mode']['parity']]
for c,x in d['configs'].items(): s=x.get('stream_mode') or {}; out += [c, round(x['ms_per_step'],3), s.get('ms_per_call'), s.get('parity')]
print(*out)" 2>&1 | tail -1
done
