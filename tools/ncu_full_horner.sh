#!/bin/bash
# ncu --set full of one Horner-step launch of a cfg5 apply (step launch 322 of prof_apply.py cfg5 1)
mkdir -p gpurun_out
timeout 300 python tools/prof_apply.py cfg5 1 > gpurun_out/plain1.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:subdomain_step -s 322 -c 1 \
  -o gpurun_out/prof_horner_r02 python tools/prof_apply.py cfg5 1 > gpurun_out/ncu_full.log 2>&1
echo rc=$? >> gpurun_out/ncu_full.log
