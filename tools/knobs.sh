#!/bin/bash
# Build timing-experiment variants of libpslr.so (csrc knobs PSLR_X_*) into lib_variants/
# and run tools/level_floor.py + a short bench against each (on the GPU box).
#   build: tools/knobs.sh build "base" "NOSTG" "XPOS" ...   run: tools/knobs.sh
set -e
cd "$(dirname "$0")/.."
mkdir -p lib_variants
if [ "$1" == "build" ]; then
  shift
  rm -f lib_variants/*.so
  for v in "$@"; do
    name=$(echo $v | tr ' ' '_')
    defs=""; for k in $v; do [ "$k" != base ] && defs="$defs -DPSLR_X_$k"; done
    touch paper_2002_00917_b200/csrc/step_kernel.cu
    make -s -C paper_2002_00917_b200/csrc EXTRA="$defs" > /dev/null 2>&1
    cp paper_2002_00917_b200/lib/libpslr.so lib_variants/libpslr_$name.so
  done
  touch paper_2002_00917_b200/csrc/step_kernel.cu; make -s -C paper_2002_00917_b200/csrc
  exit 0
fi
for f in lib_variants/libpslr_*.so; do
  n=$(basename $f .so)
  PSLR_LIB=$PWD/$f timeout 300 python bench.py --steps 200 --warmup 3 --no-cpu-baseline --e2e-steps 3 --gmres-maxit 0 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('$n bench: ms/apply %.4f' % d['ms_per_step'], {k: round(v,3) for k,v in d['roofline']['launch_ms'].items()})"
done
