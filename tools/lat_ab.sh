for v in 100000 128 64 32; do echo "NID_LAT_STEPS=$v"; NID_LAT_STEPS=$v python tools/probe_c3_levels.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()); continue
    print({k: d[k] for k in d if k in ('stage','track_ms','wall_s','endpoint_ms','steps_max','counts')})
"; done
