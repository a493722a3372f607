#!/bin/bash
# A/B the C2 headline: "new" = in-tree libivrgs.so; "old" = libivrgs_ab.so,
# or, when AB_OLD_ENV is set (e.g. AB_OLD_ENV="IVR_WORKLIST=0"), the in-tree
# library under that environment.   usage: bash tools/ab.sh [rounds]
R=${1:-2}
for i in $(seq $R); do for v in new old; do
  if [ $v = old ]; then
    if [ -n "$AB_OLD_ENV" ]; then export $AB_OLD_ENV; else export IVR_LIB_PATH=$PWD/paper_2504_17954_b200/libivrgs_ab.so; fi
  else unset IVR_LIB_PATH; [ -n "$AB_OLD_ENV" ] && unset ${AB_OLD_ENV%%=*}; fi
  python bench.py --no-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$v', round(d['value']), round(d['e2e']['value']), [round(x,3) for x in r['frame_ms_isolated_min_med_max']], {k:round(v,4) for k,v in r['stage_ms_uncaptured'].items()})"
done; done
