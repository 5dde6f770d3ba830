for r in 1 2 3; do
for v in A B; do
  if [ $v = A ]; then export ER_LIB=$PWD/paper_2605_13766_b200/lib/libA_old.so; else unset ER_LIB; fi
  python bench.py --steps 300 --no-cpu-baseline --no-e2e --no-contact --no-temporal > gpurun_out/cmp_$v.json 2>gpurun_out/cmp_$v.err; tail -n 2 gpurun_out/cmp_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/cmp_$v.json')); print('$v', d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['clocks']['sm_mhz'])"
done; done
