#!/bin/bash
# far-ring capacity sweep (PSLR_FAR_SLOTS): the bench's sweep, single stream and launch times
mkdir -p gpurun_out
for fs in ${FSS:-0 512 1024 2048 4096}; do
  echo -n "FAR_SLOTS=$fs "
  PSLR_FAR_SLOTS=$fs SBS=${SB:-46080} bash tools/sb_bench.sh 2>&1 | grep "SB "
done
