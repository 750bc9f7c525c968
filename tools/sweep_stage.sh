#!/bin/bash
# stage size / ring sweeps of the fused step kernel: single-stream and K-in-flight sweep
# usage: tools/sweep_stage.sh [extra bench args]   (e.g. --nv 1)
for cfg in "32768 4096" "24576 4096" "20480 4096" "16384 4096" "32768 2048" "24576 2048" "16384 2048"; do
  set -- $cfg
  PSLR_STAGE_BYTES=$1 PSLR_RING=$2 timeout 300 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit 0 "${@:3}" $EXTRA 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('SB=$1 W=$2', 'K=%d nv=%d ms/apply %.4f' % (d['config']['concurrency'], d['config'].get('vectors_per_call', 1), d['ms_per_step']), 'single %.3f' % d['config']['single_stream']['ms_per_apply'], flush=True)"
done
