#!/bin/bash
# block-solve timing under PSLR_DBG experiment bits (results are wrong by design)
W=${1:-cfg5}
for d in ${DBGS:-0 1 2 3}; do PSLR_DBG=$d timeout 300 python tools/time_solve.py $W; done
