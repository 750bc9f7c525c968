#!/bin/bash
# stage size / ring sweeps of the fused step kernel (bench, no CPU baseline)
for cfg in "32768 4096" "49152 4096" "40960 4096" "24576 4096" "16384 8192" "24576 8192"; do
  set -- $cfg
  PSLR_STAGE_BYTES=$1 PSLR_RING=$2 timeout 300 python bench.py --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('SB=$1 W=$2', 'ms/apply %.3f' % d['ms_per_step'], {k: round(v,3) for k,v in d['roofline']['launch_ms'].items()})"
done
