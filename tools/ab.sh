#!/bin/bash
# A/B the C2 headline: in-tree libivrgs.so ("new") vs libivrgs_ab.so ("old").
# usage: bash tools/ab.sh [rounds]
R=${1:-2}
for i in $(seq $R); do for v in new old; do
  if [ $v = old ]; then export IVR_LIB_PATH=$PWD/paper_2504_17954_b200/libivrgs_ab.so; else unset IVR_LIB_PATH; fi
  python bench.py --no-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$v', round(d['value']), round(d['e2e']['value']), [round(x,3) for x in r['frame_ms_isolated_min_med_max']], {k:round(v,4) for k,v in r['stage_ms_uncaptured'].items()})"
done; done
