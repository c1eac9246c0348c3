#!/bin/bash
# Bench one config under several env settings (experiments).  usage:
#   CFG=C2 CONFIGS=C3 bash tools/gpu_envs.sh "base:" "k1:SW_FOLD_KMIN=1" "s16:SW_SEED_N=16384,SW_FOLD_KMIN=1"
CFG=${CFG:-C2}; mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  ( IFS=','; for kv in $envs; do [ -n "$kv" ] && export "$kv"; done
    timeout 600 python bench.py --config $CFG --configs "${CONFIGS:-}" --stream-steps 0 --no-cpu-baseline --e2e-steps 1 \
      > gpurun_out/env_${name}.json 2> gpurun_out/env_${name}.err )
  python -c "
import json; d=json.load(open('gpurun_out/env_${name}.json'))
out=['$name', '$CFG', round(d['ms_per_step'],3), all(d['parity'].values()) if d['parity'] else None]
for c,v in d.get('configs',{}).items(): out += [c, round(v.get('ms_per_step',0),3), v.get('parity') and all(v['parity'].values())]
print(*out)" 2>&1 | tail -1
done
echo done
