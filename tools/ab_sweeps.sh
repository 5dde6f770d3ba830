# A/B: the library at the PDL commit (libA_old.so) vs the current one with its default sweeps
# policy and with sweeps forced on.
for r in 1 2; do
for c in cfg3 cfg4 cfg5 cfg2 cfg1; do
  echo -n "old $c: "; ER_LIB=$PWD/paper_2605_13766_b200/lib/libA_old.so timeout 150 python tools/ab_time.py $c 512 0 | tail -n 1
  echo -n "new default $c: "; timeout 150 python tools/ab_time.py $c 512 0 | tail -n 1
  echo -n "new sw128 $c: "; ER_SWEEPS=128 timeout 150 python tools/ab_time.py $c 512 0 | tail -n 1
done; done
