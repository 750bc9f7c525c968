#!/bin/bash
# programmatic dependent launch on/off x applies in flight (cfg5 concurrent sweep)
mkdir -p gpurun_out
run() {
  local label=$1; shift
  env "$@" timeout 400 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit 0 $BARGS 2>>gpurun_out/pdl.err | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$label', 'K=%d nv=%d ms/apply %.4f' % (d['config']['concurrency'], d['config'].get('vectors_per_call', 1), d['ms_per_step']), 'single %.3f' % d['config']['single_stream']['ms_per_apply'], flush=True)"
}
for k in 8 12 16; do
  BARGS="--nv 2 --streams $k" run pdl1 PSLR_PDL=1
  BARGS="--nv 2 --streams $k" run pdl0 PSLR_PDL=0
done
BARGS="--nv 1 --streams 16" run pdl0 PSLR_PDL=0
BARGS="--nv 1 --streams 8" run pdl0 PSLR_PDL=0
