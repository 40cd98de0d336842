for i in 1 2; do for o in 1 0; do TIDE_LINK_ORDERED=$o python -c "
import sys, json; sys.path.insert(0, '.')
import bench_extra as B
print('ordered=$o', [round(B.config5(t)['ms_graph'], 4) for t in (0.5, 0.7, 0.85)])"; done; done
