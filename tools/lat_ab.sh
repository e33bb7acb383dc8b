#!/bin/bash
# A/B of the per-slot evaluation threshold (TrackArgs::lat_slots) on the C3
# top probe (4,096 paths), the full C3 top and the six cascade levels.
for L in 0 4 8 12 16; do
  echo "== NID_LAT_SLOTS=$L"
  NID_LAT_SLOTS=$L python tools/probe_c3top.py 2>&1 | tail -1 | cut -c1-200
  NID_LAT_SLOTS=$L python tools/probe_c3_levels.py 2>&1 | python -c "
import sys, json
tot=0
for line in sys.stdin:
    d=json.loads(line)
    if d['stage']=='top': print('top track_ms', round(d['track_ms']), 'endpoint_ms', round(d['endpoint_ms']))
    elif d['stage'].startswith('level'):
        tot+=d['track_ms']; print(d['stage'], 'track', d['track_ms'], 'endpoint', d['endpoint_ms'], 'classify_wall', d['classify_wall_s'], d['counts'])
    elif d['stage']=='cascade total': print('cascade wall', d['wall_s'], 'track sum', round(tot))
"
done
