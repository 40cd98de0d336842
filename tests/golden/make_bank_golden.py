"""Write tests/golden/ref.bank with the REAL reference's save_bank (earlyexit 0.1.0).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bank_golden.py

A small bank (d=64, b=32, L=12, interval 4 -> checkpoints 3, 7, 11) with
seeded random routers and non-trivial stats; tests/test_bank_io.py loads it
with this package's loader and re-saves it byte for byte.
"""

import os

import numpy as np

from earlyexit import calibration as ref_cal  # from PYTHONPATH=/root/reference/pkg/src
from earlyexit.router_ops import Router

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    g = np.random.Generator(np.random.PCG64(515))
    d, b, L = 64, 32, 12
    routers, stats = {}, {}
    for i, k in enumerate(ref_cal.checkpoint_layers(L, 4, True)):
        routers[k] = Router(layer=k, w_down=(g.standard_normal((b, d)) * 0.1).astype(np.float32),
                            w_up=(g.standard_normal((1, b)) * 0.1).astype(np.float32))
        stats[k] = ref_cal.RouterStats(examples=1000 + i, positives=100 * i, final_loss=0.25 + i,
                                       accuracy=0.5 + 0.125 * i, flags=i & 1)
    bank = ref_cal.RouterBank(hidden_dim=d, bottleneck=b, interval=4, tau=0.98, eps=1e-6,
                              num_layers=L, model_digest=0x0123456789ABCDEF, routers=routers,
                              stats=stats)
    path = os.path.join(HERE, "ref.bank")
    ref_cal.save_bank(bank, path)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
