#!/bin/bash
# level-floor timing under PSLR_DBG experiment bits (results are wrong by design)
for d in 0 1 2 3; do echo "dbg=$d"; PSLR_DBG=$d timeout 120 python tools/level_floor.py 64000 32; done
