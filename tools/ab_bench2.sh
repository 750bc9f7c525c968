#!/bin/bash
# timing-only A/B/C of variant libraries against the default build (cfg5 bench)
for lib in default "$@" default "$@"; do
  if [ $lib = default ]; then unset PSLR_LIB; else export PSLR_LIB=$PWD/lib_variants/$lib/libpslr.so; fi
  timeout 400 python bench.py --steps 800 --warmup 3 --no-cpu-baseline --gmres-maxit 0 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$lib', 'ms/apply %.4f' % d['ms_per_step'], 'single %.3f' % d['config']['single_stream']['ms_per_apply'], 'e2e %.0f' % d['e2e']['value'], flush=True)"
done
unset PSLR_LIB
