#!/bin/bash
# Interleaved A/B of prebuilt libraries on the GPU box (development aid):
#   tools/ab_lib_pair.sh cfg3 300 "" lib_ab/libA.so lib_ab/libB.so ...
# Each library is timed with tools/warp_ab.py (args 1-3: config, steps, environment settings).
cfg=$1; steps=$2; envs=$3; shift 3
for r in 1 2 3; do
  for lib in "$@"; do
    echo -n "$lib: "; ER_LIB=$lib timeout 200 python tools/warp_ab.py "$cfg" "$steps" "$envs" 2>&1 | grep "rep=0"
  done
done
