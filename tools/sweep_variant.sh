#!/bin/bash
# Narrow-CTA experiment: 7 consumer warps + producer, 2 CTAs per SM (lib_variants/narrow)
# against the default 15+1-warp build, concurrent apply sweep on cfg5.
mkdir -p gpurun_out
run() {  # label, extra env..., -- bench args
  local label=$1; shift
  env "$@" timeout 400 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit 0 $BARGS 2>>gpurun_out/variant.err | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$label', 'K=%d nv=%d ms/apply %.4f' % (d['config']['concurrency'], d['config'].get('vectors_per_call', 1), d['ms_per_step']), 'single %.3f' % d['config']['single_stream']['ms_per_apply'], 'horner %.3f' % d['roofline']['launch_ms']['horner_step'], flush=True)"
}
NARROW="PSLR_LIB=$PWD/lib_variants/narrow/libpslr.so PSLR_SMEM_CAP=115712 PSLR_STAGE_BYTES=16384 PSLR_RING=2048"
PSLR_LIB=$PWD/lib_variants/narrow/libpslr.so PSLR_SMEM_CAP=115712 PSLR_STAGE_BYTES=16384 PSLR_RING=2048 \
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bitexact or multi or clones" > gpurun_out/variant_pytest.log 2>&1
tail -1 gpurun_out/variant_pytest.log
BARGS="--nv 2" run wide_nv2 A=1
BARGS="--nv 1" run wide_nv1 A=1
for k in 8 9; do
  BARGS="--nv 2 --streams $k" run narrow_nv2_K$k $NARROW
  BARGS="--nv 1 --streams $k" run narrow_nv1_K$k $NARROW
done
BARGS="--nv 1 --streams 16" run narrow_nv1_K16 $NARROW
BARGS="--nv 2 --streams 8" run wide_sb16_r2048 PSLR_STAGE_BYTES=16384 PSLR_RING=2048
