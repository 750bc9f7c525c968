#!/bin/bash
# Two step CTAs per SM (7 consumer warps, <= 113 KB shared memory each) in the concurrent
# sweep: variant library lib_variants/t224m2 (PSLR_STEP_THREADS=224, PSLR_STEP_MINB=2).
mkdir -p gpurun_out
run() {  # label, env..., -- bench args
  local label=$1; shift
  echo -n "$label: "
  env "$@" timeout 400 python bench.py --steps 400 --warmup 3 --no-cpu-baseline --e2e-steps 8 --gmres-maxit 0 --solves "" $BARGS 2>>gpurun_out/occ2.err | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    c=d['config']
    print('ms/apply %.4f' % d['ms_per_step'], 'nv', c['vectors_per_call'], 'streams', c['concurrency'], 'single %.3f' % c['single_stream']['ms_per_apply'], flush=True)"
}
V=$PWD/lib_variants/t224m2/libpslr.so
BARGS="" run default PSLR_X=0
BARGS="--streams 32" run default_s32 PSLR_X=0
BARGS="--streams 32" run t224_nv2_sb16 PSLR_LIB=$V PSLR_SMEM_CAP=115712 PSLR_STAGE_BYTES2=16384 PSLR_STAGE_BYTES=24576
BARGS="--streams 32" run t224_nv2_w2048 PSLR_LIB=$V PSLR_SMEM_CAP=115712 PSLR_RING=2048 PSLR_STAGE_BYTES2=24576 PSLR_STAGE_BYTES=24576
BARGS="--streams 32 --nv 1" run t224_nv1 PSLR_LIB=$V PSLR_SMEM_CAP=115712 PSLR_STAGE_BYTES=24576
BARGS="--streams 48 --nv 1" run t224_nv1_s48 PSLR_LIB=$V PSLR_SMEM_CAP=115712 PSLR_STAGE_BYTES=24576
BARGS="--streams 16 --nv 1" run default_nv1 PSLR_X=0
