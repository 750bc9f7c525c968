#!/bin/bash
# GPU check: parity tests, the N=1 bench line (short), the sharded native path on one rank, the reference arm
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 200 --warmup 3 --gmres-maxit 100 --cpu-applies 1 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --sharded --steps 64 --warmup 3 --gmres-maxit 50 > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err; echo "rc=$?" >> gpurun_out/bench_sharded.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
echo done
