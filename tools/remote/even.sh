for i in 1 2; do for e in 0 1; do TIDE_K1M_EVEN=$e python -c "
import sys; sys.path.insert(0, '.')
import bench_extra as B
print('even=$e', [round(B.config2(t)['ms_graph'], 4) for t in (0.5, 1.0)], round(B.config5(1.0)['ms_graph'], 4))"; done; done
timeout 300 python -m pytest tests/test_gpu_posthoc.py -q -p no:cacheprovider -k "multi or spec or odd or repeats" 2>&1 | tail -1
