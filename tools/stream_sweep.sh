#!/bin/bash
timeout 60 python tools/time_solve.py cfg5; timeout 60 python tools/time_solve.py 1d
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
