#!/bin/bash
# stage size x stage count of the one-vector plan on the cfg5 block solves (late round 2):
# solve_B full (dbg=0) and the stream alone (dbg=16); the far-ring takes what the stages leave
mkdir -p gpurun_out
export PSLR_SETUP_CACHE=/tmp/pslr_cache PSLR_MERGE=${PSLR_MERGE:-2}
CFGS=${CFGS:-53248,3 46080,3 40960,3 36864,4 32768,4 32768,5 28672,5 26624,6 24576,6 20480,7 18432,8}
for cfg in $CFGS; do
  sb=${cfg%,*}; ns=${cfg#*,}
  for d in ${DBGS:-0 16}; do
    echo -n "SB=$sb stages=$ns: "
    PSLR_STAGE_BYTES=$sb PSLR_MAX_STAGES=$ns PSLR_DBG=$d timeout 200 python tools/time_solve.py ${WL:-cfg5} 2>&1 | grep "dbg=" || echo failed
  done
done
