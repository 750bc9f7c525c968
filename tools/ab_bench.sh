#!/bin/bash
# timing-only A/B of a variant library (no parity tests: for experiments whose results are
# deliberately wrong, e.g. a store-order upper bound)
V=$1
for lib in default $V default $V; do
  if [ $lib = default ]; then unset PSLR_LIB; else export PSLR_LIB=$PWD/lib_variants/$V/libpslr.so; fi
  timeout 400 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --gmres-maxit 0 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    L=d['roofline']['launch_ms']
    print('$lib', 'ms/apply %.4f' % d['ms_per_step'], 'single %.3f' % d['config']['single_stream']['ms_per_apply'], 'first %.3f horner %.3f last %.3f' % (L['first_step'], L['horner_step'], L['last_step']), flush=True)"
done
unset PSLR_LIB
