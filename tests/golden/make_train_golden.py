"""Write tests/golden/train.npz with the REAL reference's train_router (earlyexit 0.1.0).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_train_golden.py

Each case regenerates its features / labels from a seed (TRAIN_CASES below,
shared with tests/test_gpu_training.py) and stores the trained w_down, w_up
and RouterStats fields.
"""

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# name -> (seed, n, d, label column, feature scale of column 0, config kwargs)
TRAIN_CASES = {
    "separable_d64": (3, 2000, 64, 0, 1.0,
                      dict(epochs=60, seed=5, learning_rate=1e-2, batch_size=128)),
    "short_d16": (11, 300, 16, 1, 1.0, dict(epochs=5, seed=9)),
    "margin_d256": (404, 3000, 256, 0, 4.0,
                    dict(epochs=8, seed=7, learning_rate=1e-3, batch_size=256)),
    "ragged_batches_d96": (21, 1000, 96, 2, 1.0,
                           dict(epochs=4, seed=2, learning_rate=3e-3, batch_size=384,
                                bottleneck=40)),
}


def case_data(name):
    seed, n, d, col, scale, _ = TRAIN_CASES[name]
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((n, d), dtype=np.float32)
    x[:, col] *= np.float32(scale)
    y = (x[:, col] > 0).astype(np.float32)
    return x, y


def main():
    from earlyexit.calibration import CalibrationConfig, train_router  # the reference

    out = {}
    for name, (_, _, _, _, _, kw) in TRAIN_CASES.items():
        x, y = case_data(name)
        r, st = train_router(x, y, layer=3, config=CalibrationConfig(**kw))
        out[f"{name}__w_down"] = r.w_down
        out[f"{name}__w_up"] = r.w_up
        out[f"{name}__stats"] = np.array([st.examples, st.positives, st.final_loss, st.accuracy,
                                          st.flags], np.float64)
    np.savez_compressed(os.path.join(HERE, "train.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
