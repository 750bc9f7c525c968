#!/bin/bash
# One GPU session: tests, smoke, bench (default), launch list + full ncu capture of a Horner launch.
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 300 python tools/prof_apply.py cfg5 3 > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_apply.py cfg5 3 > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_apply.py cfg5 1 > gpurun_out/plain1.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "pslr_apply/" -k regex:subdomain_step -s 2 -c 1 -o gpurun_out/prof_horner python tools/prof_apply.py cfg5 1 > gpurun_out/ncu_full.log 2>&1
echo done
