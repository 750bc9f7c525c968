#!/bin/bash
# stream rate vs stage plan: solve_B / solve_C0 on cfg5 (full and stream-only, dbg=16)
mkdir -p gpurun_out
run() { echo "== $*"; for d in 0 16; do env "$@" PSLR_DBG=$d timeout 200 python tools/time_solve.py cfg5 2>&1 | grep cfg5; done; }
run A=default
run PSLR_LIB=$PWD/lib_variants/cr512/libpslr.so
run PSLR_LIB=$PWD/lib_variants/cr512/libpslr.so PSLR_STAGE_BYTES=24576
run PSLR_LIB=$PWD/lib_variants/cr256/libpslr.so PSLR_STAGE_BYTES=16384
run PSLR_LIB=$PWD/lib_variants/cr256/libpslr.so PSLR_STAGE_BYTES=20480
run PSLR_LIB=$PWD/lib_variants/cr512/libpslr.so PSLR_RING=2048
