#!/bin/bash
# A/B of variant libraries on the cfg5 block solves: full and stream-only (dbg=16)
# usage: tools/ab_solve.sh name1 name2 ...   (default = the in-tree build)
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then unset PSLR_LIB; else export PSLR_LIB=$PWD/lib_variants/$v/libpslr.so; fi
  for d in ${DBGS:-0 16}; do echo -n "$v: "; PSLR_DBG=$d timeout 200 python tools/time_solve.py ${WL:-cfg5} 2>&1 | grep dbg; done
done
unset PSLR_LIB
