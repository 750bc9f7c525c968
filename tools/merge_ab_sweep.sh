set -x
for w in 240 480 720; do PSLR_MERGE_W=$w MODES=0,3 timeout 300 python tools/merge_ab.py cfg5; done
PSLR_MERGE_W=480 MODES=3 timeout 300 python tools/merge_ab.py cfg2 cfg3
