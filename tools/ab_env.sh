#!/bin/bash
# A/B one environment switch on the GPU box: tools/ab_env.sh VAR=value cfg steps  (A = unset)
for r in 1 2; do
  echo -n "A: "; timeout 150 python tools/ab_time.py "$2" "$3" 0 | tail -1
  echo -n "B ($1): "; env "$1" timeout 150 python tools/ab_time.py "$2" "$3" 0 | tail -1
done
