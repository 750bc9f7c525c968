#!/bin/bash
# stage-size sweep through the bench: concurrent sweep ms/apply, single stream, Horner launch
mkdir -p gpurun_out
for sb in ${SBS:-53248}; do
  PSLR_STAGE_BYTES=$sb timeout 400 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit 0 --solves "" 2>>gpurun_out/sb_bench.err | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    L=d['roofline']['launch_ms']
    print('SB $sb', 'sweep ms/apply %.4f' % d['ms_per_step'], 'single %.3f' % d['config']['single_stream']['ms_per_apply'], ' '.join('%s %.1f' % (k, v*1e3) for k, v in L.items()), flush=True)"
done
