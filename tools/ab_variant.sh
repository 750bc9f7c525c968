#!/bin/bash
# A/B of a variant library (lib_variants/$1) against the default build: GPU parity tests
# under the variant, then the cfg5 bench (concurrent sweep + single-stream latency).
V=$1
mkdir -p gpurun_out
PSLR_LIB=$PWD/lib_variants/$V/libpslr.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x > gpurun_out/ab_${V}_pytest.log 2>&1
tail -1 gpurun_out/ab_${V}_pytest.log
for lib in default $V default $V; do
  if [ $lib = default ]; then unset PSLR_LIB; else export PSLR_LIB=$PWD/lib_variants/$V/libpslr.so; fi
  timeout 400 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit 0 2>>gpurun_out/ab.err | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    L=d['roofline']['launch_ms']
    print('$lib', 'ms/apply %.4f' % d['ms_per_step'], 'single %.3f' % d['config']['single_stream']['ms_per_apply'], 'first %.3f horner %.3f last %.3f corr_c0 %.3f' % (L['first_step'], L['horner_step'], L['last_step'], L['correction_c0']), flush=True)"
done
unset PSLR_LIB
