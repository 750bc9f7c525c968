#!/bin/bash
for d in 0 16; do echo "== dbg=$d"; PSLR_DBG=$d PSLR_LIB=$PWD/lib_variants/trace1/libpslr.so PSLR_TRACE=1 timeout 200 python tools/trace_apply.py cfg5 2>&1 | grep -A5 "per CTA"; done
