timeout 900 python -m pytest tests/test_gpu_compact_project.py tests/test_gpu_route.py tests/test_gpu_labels.py tests/test_gpu_reference_suite.py -q -p no:cacheprovider --tb=short 2>&1 | tail -4
python -c "
import sys; sys.path.insert(0, '.')
import bench_extra as B; print(B.dropin_numpy())"
python -c "
import os; print('cpus', os.cpu_count()); import torch; print('torch threads', torch.get_num_threads())"
