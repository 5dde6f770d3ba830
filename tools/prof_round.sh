#!/bin/bash
# Evidence for one kernel version (GPU box).  gpurun copies back <= 64 MiB, so the ncu captures are
# separate calls:
#   tools/prof_round.sh <out_dir> bench          smoke, bench JSON of cfg1-cfg5, ncu launch list
#   tools/prof_round.sh <out_dir> <cfg> <regex>  one full ncu capture of that config's step kernel
set -x
out=$1; what=$2
mkdir -p $out
if [ "$what" = bench ]; then
  python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
  python bench.py > $out/bench.json 2> $out/bench.err
  for c in cfg4 cfg5 cfg2 cfg1; do
    python bench.py --config $c --no-cpu-fanout --no-contact --no-e2e > $out/bench_$c.json 2> $out/bench_$c.err
  done
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-temporal --no-contact > $out/ncu_launch.log 2>&1
else
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o $out/${what}_full \
    python tools/prof_run.py $what 1 5 > $out/ncu_$what.log 2>&1
fi
ls -la $out
