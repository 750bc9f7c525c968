#!/bin/bash
for d in ${DBGS:-768 0}; do
  PSLR_DBG=$d timeout 200 python bench.py --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('DBG=$d', 'ms/apply %.3f' % d['ms_per_step'], {k: round(v,3) for k,v in d['roofline']['launch_ms'].items()})"
done
