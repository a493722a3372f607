#!/bin/bash
# C2 headline under several builds of libivrgs, interleaved.
# usage: bash tools/ab_libs.sh rounds lib_a.so lib_b.so ...   ("-" = in-tree build)
R=$1; shift
for i in $(seq $R); do for l in "$@"; do
  if [ "$l" = "-" ]; then unset IVR_LIB_PATH; else export IVR_LIB_PATH=$PWD/$l; fi
  python bench.py --no-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$l', round(d['value']), round(d['e2e']['value']), [round(x,3) for x in r['frame_ms_isolated_min_med_max']], {k:round(v,4) for k,v in r['stage_ms_uncaptured'].items()})"
done; done
