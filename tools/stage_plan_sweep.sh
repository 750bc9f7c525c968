#!/bin/bash
# stage count of the one- and two-vector plans (the far-ring takes what the stages leave)
for s1 in ${S1S:-3 4}; do for s2 in ${S2S:-3 4}; do
  echo -n "stages1=$s1 stages2=$s2 "
  PSLR_MAX_STAGES=$s1 PSLR_MAX_STAGES2=$s2 SBS=46080 bash tools/sb_bench.sh 2>&1 | grep "SB "
done; done
