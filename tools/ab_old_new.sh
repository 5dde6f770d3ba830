# A/B of the current library against paper_2605_13766_b200/lib/libA_old.so (build it from another
# commit first: git stash; python paper_2605_13766_b200/build.py --force; cp .../libelasticarod.so .../libA_old.so; git stash pop)
for cfg in cfg3 cfg4 cfg5 fibres; do
  for r in 1 2; do
    echo -n "old $cfg: "; ER_LIB=$PWD/paper_2605_13766_b200/lib/libA_old.so timeout 150 python tools/ab_time.py $cfg 300 0 | tail -1
    echo -n "new $cfg: "; timeout 150 python tools/ab_time.py $cfg 300 0 | tail -1
  done
done
