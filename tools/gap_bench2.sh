# Same with sweeps forced (few launches, all queued up front): host-side or GPU-side stall?
for r in 1 2 3 4; do
  for sw in 1 128; do
    ER_BENCH_CLOCK_MS=100 python bench.py --config cfg4 --sweeps $sw --no-cpu-baseline --no-e2e --no-contact --no-temporal > gpurun_out/gb.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/gb.json')); r=d['roofline']; print('sweeps=$sw', round(d['ms_per_step'],4), round(r['kernel_ms_per_launch'],4), round(r['kernel_share_of_step'],3), d['clocks']['samples'], d['gpu_launches'])"
  done
done
