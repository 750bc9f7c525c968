#!/bin/bash
# per-level cost vs width (trace build 3) on the deepest cfg5 blocks and block 1 (wide L)
mkdir -p gpurun_out
for cta in 23 19 1; do
  PSLR_LIB=$PWD/lib_variants/trace3/libpslr.so PSLR_TRACE=1 PSLR_TRACE_CTA=$cta timeout 300 python tools/trace_levels.py cfg5 B >> gpurun_out/trace_levels.log 2>&1
done
for cta in 23 19; do
  PSLR_LIB=$PWD/lib_variants/trace3/libpslr.so PSLR_TRACE=1 PSLR_TRACE_CTA=$cta timeout 300 python tools/trace_levels.py cfg5 C0 >> gpurun_out/trace_levels.log 2>&1
done
timeout 300 python tools/time_solve.py cfg5 >> gpurun_out/trace_levels.log 2>&1
echo done
