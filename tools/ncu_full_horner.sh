#!/bin/bash
# ncu --set full of the first Horner step's B launch of a cfg5 apply (NVTX range pslr_apply:
# step launches first-B, correction-C0, Horner1-B, ... -> skip 2)
mkdir -p gpurun_out
timeout 300 python tools/prof_apply.py cfg5 1 > gpurun_out/plain1.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "pslr_apply/" \
  -k regex:subdomain_step -s 2 -c 1 -o gpurun_out/prof_horner_r02 python tools/prof_apply.py cfg5 1 > gpurun_out/ncu_full.log 2>&1
echo rc=$? >> gpurun_out/ncu_full.log
