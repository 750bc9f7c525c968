#!/bin/bash
# ring size W x stage bytes: single-stream latency and the concurrent sweep (cfg5)
mkdir -p gpurun_out
run() {
  local label=$1; shift
  env "$@" timeout 400 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit 0 $BARGS 2>>gpurun_out/ring2.err | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$label', 'K=%d nv=%d ms/apply %.4f' % (d['config']['concurrency'], d['config'].get('vectors_per_call', 1), d['ms_per_step']), 'single %.3f' % d['config']['single_stream']['ms_per_apply'], 'horner %.3f' % d['roofline']['launch_ms']['horner_step'], flush=True)"
}
BARGS="--nv 2" run W4096_SB32K A=1
BARGS="--nv 2" run W8192_SB32K PSLR_RING=8192
BARGS="--nv 1" run W8192_SB32K PSLR_RING=8192
BARGS="--nv 2" run W8192_SB24K PSLR_RING=8192 PSLR_STAGE_BYTES=24576
BARGS="--nv 2" run W8192_SB16K PSLR_RING=8192 PSLR_STAGE_BYTES=16384
BARGS="--nv 2" run W16384_SB16K PSLR_RING=16384 PSLR_STAGE_BYTES=16384
