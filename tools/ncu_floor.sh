#!/bin/bash
# ncu source-level capture of one solve_B launch of the 1D-chain level-floor workload
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:subdomain_step -s 3 -c 1 \
  -o gpurun_out/floor python tools/level_floor.py 64000 32 > gpurun_out/ncu_floor.log 2>&1
echo rc=$? >> gpurun_out/ncu_floor.log
