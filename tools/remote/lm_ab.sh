# A/B of two builds of the LM head (tools/_libs/lm_old vs lm_new), interleaved rounds
L=paper_2603_21365_b200/_lib
for r in 0 1 2; do
  for v in old new; do
    cp tools/_libs/lm_$v/libtide_b200.so tools/_libs/lm_$v/build.stamp $L/
    TIDE_ALLOW_STALE=1 python -c "
import sys; sys.path.insert(0, '.')
import bench_extra as B; x = B.lm_head()
print('$v', f\"3term {x['ms_3term']:.3f} ms 1term {x['ms_1term_bf16']:.3f} ms\")" 2>&1 | tail -1
  done
done
cp tools/_libs/lm_new/libtide_b200.so tools/_libs/lm_new/build.stamp $L/
timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -p no:cacheprovider 2>&1 | tail -2
