#!/bin/bash
# Evidence for one kernel version (GPU box): bench JSON for the configs, the ncu launch list of the
# bench command and one full ncu capture of the top kernel.  tools/prof_round.sh <out_dir> <kernel regex>
set -x
out=$1; kre=$2
mkdir -p $out
python bench.py > $out/bench.json 2> $out/bench.err
for c in cfg4 cfg5 cfg2 cfg1; do
  python bench.py --config $c --no-cpu-fanout --no-contact --no-e2e > $out/bench_$c.json 2> $out/bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-temporal --no-contact > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$kre -s 3 -c 1 -o $out/top_full \
  python tools/prof_run.py cfg3 1 5 > $out/ncu_full.log 2>&1
ls -la $out
