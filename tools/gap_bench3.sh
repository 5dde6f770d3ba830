# Gaps between step launches under clock sampling: nvidia-smi process vs in-process NVML (cfg4).
for r in 1 2 3 4; do
  for mode in nvml smi; do
    ER_BENCH_CLOCKS=$mode python bench.py --config cfg4 --no-cpu-baseline --no-e2e --no-contact --no-temporal > gpurun_out/gb.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/gb.json')); r=d['roofline']; print('$mode', round(d['ms_per_step'],4), round(r['kernel_ms_per_launch'],4), round(r['kernel_share_of_step'],3), d['clocks'])"
  done
done
