# Gaps between step launches under clock sampling: WHILE step graph (default) vs one graph
# launch per 32 steps (ER_NO_WHILE_GRAPH=1), cfg4 and cfg3.
for r in 1 2 3; do
  for c in cfg4 cfg3; do
    for mode in while plain; do
      if [ $mode = plain ]; then export ER_NO_WHILE_GRAPH=1; else unset ER_NO_WHILE_GRAPH; fi
      python bench.py --config $c --no-cpu-baseline --no-e2e --no-contact --no-temporal > gpurun_out/gb.json 2>/dev/null
      python -c "
import json; d=json.load(open('gpurun_out/gb.json')); r=d['roofline']; print('$c $mode', round(d['ms_per_step'],4), round(r['kernel_ms_per_launch'],4), round(r['kernel_share_of_step'],3), d['clocks']['sm_mhz'], d['gpu_launches'])"
    done
  done
done
