# cfg3 in the bench setting (clock sampler on): one launch per step (WHILE step graph) vs 128
# sweeps per launch, alternating.
for r in 1 2 3 4 5; do
  for sw in 1 128; do
    python bench.py --sweeps $sw --no-cpu-baseline --no-e2e --no-contact --no-temporal > gpurun_out/gb.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/gb.json')); r=d['roofline']; print('sweeps=$sw', round(d['ms_per_step'],4), round(r['kernel_ms_per_launch'],4), round(r['kernel_share_of_step'],3), d['clocks']['sm_mhz'])"
  done
done
