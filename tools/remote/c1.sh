for e in "" "TIDE_F32_TAIL_ROWS=0" "TIDE_F32_TAIL_ROWS=0 TIDE_F32_TC=1"; do env $e python -c "
import sys; sys.path.insert(0, '.')
import bench_extra as B
r = B.config1(); print('$e', round(r['ms_graph'], 4), round(r['ms_api'], 4))"; done
