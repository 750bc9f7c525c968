#!/bin/bash
# ring size x stage size sweep, NV = 1 and 2 per call (bench sweep, 8 calls in flight)
for nv in 2 1; do
for cfg in "32768 4096" "32768 8192" "24576 8192" "16384 8192" "12288 8192"; do
  set -- $cfg
  PSLR_STAGE_BYTES=$1 PSLR_RING=$2 timeout 300 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit 0 --nv $nv 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('SB=$1 W=$2', 'K=%d nv=%d ms/apply %.4f' % (d['config']['concurrency'], d['config'].get('vectors_per_call', 1), d['ms_per_step']), 'single %.3f' % d['config']['single_stream']['ms_per_apply'], 'horner %.3f' % d['roofline']['launch_ms']['horner_step'], flush=True)"
done; done
