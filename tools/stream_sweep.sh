#!/bin/bash
timeout 120 python tools/time_solve.py cfg5; timeout 120 python tools/time_solve.py 1d
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contract.py -q -x 2>&1 | tail -2
