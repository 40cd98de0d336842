timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -p no:cacheprovider -x 2>&1 | tail -3
TIDE_LM_PAIR=0 timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -p no:cacheprovider -x 2>&1 | tail -1
python -c "
import sys, json; sys.path.insert(0, '.')
import bench_extra as B
print(json.dumps(B.lm_head()))"
TIDE_LM_PAIR=0 python -c "
import sys, json; sys.path.insert(0, '.')
import bench_extra as B
print(json.dumps(B.lm_head()))"
