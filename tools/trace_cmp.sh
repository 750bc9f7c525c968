#!/bin/bash
# per-level cost vs width, two trace builds (default 480 consumer threads vs 256), CTA 19
mkdir -p gpurun_out
for v in trace3 trace3_t256; do echo "== $v"; PSLR_LIB=$PWD/lib_variants/$v/libpslr.so PSLR_TRACE=1 PSLR_TRACE_CTA=19 timeout 300 python tools/trace_levels.py cfg5 B; done
