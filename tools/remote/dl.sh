timeout 900 python -m pytest tests/test_gpu_compact_project.py tests/test_gpu_lmhead.py tests/test_gpu_labels.py tests/test_gpu_reference_suite.py -q -p no:cacheprovider --tb=short 2>&1 | tail -4
python - <<'PY'
import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2603_21365_b200 as P
from paper_2603_21365_b200 import _device as D
t = torch.randn(4096, 50260, device='cuda')
for f, name in ((lambda: t.cpu().numpy(), 'pageable'), (lambda: D.to_host(t), 'staged')):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): f()
    dt = (time.perf_counter() - t0) / 5
    print(name, f"{dt*1e3:.1f} ms  {t.numel()*4/dt/1e9:.1f} GB/s")
PY
