#!/bin/bash
# stage size sweep of the fused step kernel: 8-in-flight sweep (nv 2 and 1) + single-stream latency
# usage: tools/sweep_stage.sh "SB1 SB2 ..." [ring]
SBS=${1:-"32768 40960 49152 65536"}
RING=${2:-4096}
for nv in 2 1; do
for sb in $SBS; do
  PSLR_STAGE_BYTES=$sb PSLR_RING=$RING timeout 300 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit 0 --nv $nv 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('SB=$sb W=$RING', 'K=%d nv=%d ms/apply %.4f' % (d['config']['concurrency'], d['config'].get('vectors_per_call', 1), d['ms_per_step']), 'single %.3f' % d['config']['single_stream']['ms_per_apply'], 'horner %.3f' % d['roofline']['launch_ms']['horner_step'], flush=True)"
done; done
