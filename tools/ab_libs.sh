#!/bin/bash
# A/B two builds of the library on the GPU box: tools/ab_libs.sh "<nvcc extra flags for B>" cfg steps
# (A = the default build).  Runs interleaved, 3 rounds each.
set -e
python paper_2605_13766_b200/build.py --force > /dev/null 2>&1
cp paper_2605_13766_b200/lib/libelasticarod.so /tmp/libA.so
ER_NVCC_EXTRA="$1" python paper_2605_13766_b200/build.py --force > /dev/null 2>&1
cp paper_2605_13766_b200/lib/libelasticarod.so /tmp/libB.so
for r in 1 2 3; do
  for v in A B; do
    echo -n "$v: "; ER_LIB=/tmp/lib$v.so timeout 120 python tools/ab_time.py "$2" "$3" 0 | tail -1
  done
done
