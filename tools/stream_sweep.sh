#!/bin/bash
L=$PWD/lib_variants
for v in default pre8_8 pre16_8 default pre8_8 pre16_8; do
  if [ $v = default ]; then unset PSLR_LIB; else export PSLR_LIB=$L/$v/libpslr.so; fi
  echo -n "$v "; timeout 120 python tools/time_solve.py cfg5
done
