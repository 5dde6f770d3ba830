# Does the clock sampler (nvidia-smi -lms) open gaps between step launches?  cfg4, three settings.
for r in 1 2 3; do
  for mode in sampler100 nosampler sampler500; do
    case $mode in
      sampler100) env="ER_BENCH_CLOCK_MS=100";;
      nosampler) env="ER_BENCH_NO_CLOCKS=1";;
      sampler500) env="ER_BENCH_CLOCK_MS=500";;
    esac
    env $env python bench.py --config cfg4 --no-cpu-baseline --no-e2e --no-contact --no-temporal > gpurun_out/gb.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/gb.json')); r=d['roofline']; print('$mode', round(d['ms_per_step'],4), round(r['kernel_ms_per_launch'],4), round(r['kernel_share_of_step'],3), d['clocks']['samples'])"
  done
done
