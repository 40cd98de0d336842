bash tools/remote/lm_ab.sh
for v in old new; do
  cp tools/_libs/lm_$v/libtide_b200.so tools/_libs/lm_$v/build.stamp paper_2603_21365_b200/_lib/
  TIDE_ALLOW_STALE=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:lmhead2p -c 1 python -c "
import sys; sys.path.insert(0, '.')
import bench_extra as B; B.lm_head()" 2>&1 | grep -E "dram__bytes|duration" | sed "s/^/$v /"
done
cp tools/_libs/lm_new/libtide_b200.so tools/_libs/lm_new/build.stamp paper_2603_21365_b200/_lib/
