#!/bin/bash
# one CTA alone (its stream has HBM to itself) vs the full grid: is the factor stream
# the bound of the level loop on cfg5?
mkdir -p gpurun_out
for b in -1 19 23 1; do for d in 0 16 1; do echo -n "block $b: "; PSLR_ONLY_BLOCK=$b PSLR_DBG=$d timeout 200 python tools/time_solve.py cfg5 2>&1 | grep dbg; done; done
