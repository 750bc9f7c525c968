#!/bin/bash
# A/B of environment settings on the cfg5 bench (sweep, single stream, per-launch times):
# usage: tools/ab_env.sh "label1:VAR=a VAR2=b" "label2:VAR=c" ...   (two rounds, interleaved)
mkdir -p gpurun_out
export PSLR_SETUP_CACHE=${PSLR_SETUP_CACHE:-/tmp/pslr_cache}
for rep in 1 2; do
for spec in "$@"; do
  label=${spec%%:*}; envs=${spec#*:}
  env $envs timeout 400 python bench.py --steps ${STEPS:-200} --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit ${GMRES_MAXIT:-0} --solves "" 2>>gpurun_out/ab.err | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    L=d['roofline']['launch_ms']
    g=[s for s in d.get('solves',[]) if s['config']=='cfg5']
    print('$label', 'ms/apply %.4f' % d['ms_per_step'], 'single %.3f' % d['config']['single_stream']['ms_per_apply'], 'first %.3f horner %.3f last %.3f corr_c0 %.3f' % (L['first_step'], L['horner_step'], L['last_step'], L['correction_c0']), ('gmres %.3f ms/it' % g[0]['ms_per_iteration']) if g else '', flush=True)"
done; done
