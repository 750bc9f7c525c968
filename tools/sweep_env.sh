#!/bin/bash
# bench under several environment settings: sweep_env.sh "A=1 B=2" "A=0" ...
for e in "$@"; do
  env $e timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 3 --gmres-maxit 0 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('$e', 'ms/apply %.4f' % d['ms_per_step'], {k: round(v,3) for k,v in d['roofline']['launch_ms'].items()})"
done
