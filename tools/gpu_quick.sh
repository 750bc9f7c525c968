#!/bin/bash
# Quick GPU iteration: gpu tests (stop at first failure) + a short bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline --gmres-maxit ${GMRES_MAXIT:-100} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
echo done
