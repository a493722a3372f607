#!/bin/bash
# C2 headline under several environments, interleaved.
# usage: bash tools/ab_env.sh rounds "ENV_A" "ENV_B" ...   ("-" = no extra env)
R=$1; shift
for i in $(seq $R); do for e in "$@"; do
  if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
  env $envs python bench.py --no-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$e', round(d['value']), round(d['e2e']['value']), [round(x,3) for x in r['frame_ms_isolated_min_med_max']], {k:round(v,4) for k,v in r['stage_ms_uncaptured'].items()})"
done; done
