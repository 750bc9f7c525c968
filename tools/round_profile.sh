#!/bin/bash
# Round profiling (one GPU): per-launch time + DRAM bytes of cfg5 applies (one and two
# vectors per call), a full ncu capture of one Horner-step launch, and the bench's own
# launch list.  Summarised here by tools/ncu_summary_r02.py into profiles/.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 python tools/prof_apply.py cfg5 2 > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_nv1.csv python tools/prof_apply.py cfg5 2 > gpurun_out/ncu_nv1.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_nv2.csv python tools/prof_apply.py cfg5 2 2 > gpurun_out/ncu_nv2.log 2>&1
# the Horner launches of the applies: skip the build's step launches (Arnoldi: rank x (m+2) + the C0 solves)
timeout 1200 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "pslr_apply/" -k regex:subdomain_step -s 2 -c 1 \
  -o gpurun_out/prof_horner_r02 python tools/prof_apply.py cfg5 1 > gpurun_out/ncu_full.log 2>&1
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --gmres-maxit 0 --e2e-steps 8 --solves "" > gpurun_out/b_plain.json 2>/dev/null && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/bench_launches.csv \
  python bench.py --steps 8 --warmup 3 --no-cpu-baseline --gmres-maxit 0 --e2e-steps 8 --solves "" > gpurun_out/bench_ncu.log 2>&1
echo done
