for a in "--config 5" "--config 5 --scaling strong" "--config 4" ; do
  timeout 600 python bench.py $a --steps 10 --warmup 3 2>&1 | tail -c 1300; echo
done
timeout 900 python bench_extra.py sweep 2>&1 | tail -8
