#!/bin/bash
# ncu source-level capture of one cfg5 solve_B launch (time_solve.py's 4th launch)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:subdomain_step -s 4 -c 1 \
  -o gpurun_out/solveb python tools/time_solve.py cfg5 > gpurun_out/ncu_solveb.log 2>&1
echo rc=$? >> gpurun_out/ncu_solveb.log
