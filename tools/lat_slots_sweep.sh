#!/bin/bash
# C3 step (top / cascade / filter seconds) against the per-slot threshold NID_LAT_SLOTS
for v in 2 4 6 8 12 16; do
  NID_LAT_SLOTS=$v python bench.py --workload c3 --steps 2 --warmup 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print('lat_slots $v', round(d['ms_per_step']), round(c['top_s'],3), round(c['cascade_s'],3), round(c['filter_s'],3))"
done
