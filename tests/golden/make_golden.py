"""Generate golden vectors from the REAL reference (earlyexit 0.1.0).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs are regenerated in the tests from the recorded PCG64 seeds; each
fixture stores a SHA-1 of its inputs so a numpy bit-stream change is caught
instead of silently comparing different data.  Outputs are whatever the
reference returned — they pin `oracle/tide_oracle.py` (see
tests/test_oracle_golden.py) and the GPU kernels (tests/test_gpu_*.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests.golden.cases import (LABEL_CASES, ROUTE_CASES, digest,  # noqa: E402
                                make_label_inputs, make_route_inputs, posthoc_states,
                                rigged_router_arrays)

import earlyexit  # noqa: E402  (from PYTHONPATH=/root/reference/pkg/src)
from earlyexit import calibration as ref_cal  # noqa: E402
from earlyexit import router_ops as ref_ops  # noqa: E402
from earlyexit import runtime as ref_rt  # noqa: E402
from earlyexit import tensor_math as ref_tm  # noqa: E402
from earlyexit.fixtures import make_rigged_bank  # noqa: E402


def gen_route():
    out = {}
    for name, spec in ROUTE_CASES.items():
        h, w_down, w_up = make_route_inputs(spec)
        router = ref_ops.Router(layer=3, w_down=w_down, w_up=w_up)
        fused = ref_ops.fused_layernorm_route(h, router)
        composed = ref_ops.route_scores(h, router)
        out[f"{name}__digest"] = np.frombuffer(digest(h, w_down, w_up).encode(), np.uint8)
        out[f"{name}__fused"] = fused
        out[f"{name}__composed"] = composed
    return out


def gen_compact():
    rng = np.random.Generator(np.random.PCG64(707))   # test_acceptance.py:169
    out = {}
    rows8 = rng.standard_normal((8, 5), dtype=np.float32)
    out["rows8"] = rows8
    masks = []
    for n in list(range(1, 81)) + [1000, 1000, 1000, 4097]:
        m = rng.random(n) < rng.random()
        masks.append(m)
    for i, m in enumerate(masks):
        h = np.arange(m.shape[0] * 3, dtype=np.float32).reshape(-1, 3)
        for strategy in ("small", "prefix"):
            r = ref_ops.batch_compact(h, m, strategy=strategy)
            out[f"m{i}__mask"] = m
            out[f"m{i}__{strategy}__exit"] = r.exiting_indices
            out[f"m{i}__{strategy}__cont"] = r.continuing_indices
    out["n_masks"] = np.array([len(masks)])
    return out


def gen_projection():
    rng = np.random.Generator(np.random.PCG64(99))
    gain = rng.standard_normal(64, dtype=np.float32)
    rows = rng.standard_normal((7, 64), dtype=np.float32) * 3
    positions = np.array([0, 2, 3, 9, 10, 15, 19], dtype=np.int64)
    got = np.full((20, 64), -1.0, np.float32)
    ref_ops.exit_projection(rows, gain, ref_tm.DEFAULT_EPS, positions, got)
    got_nogain = np.full((20, 64), -1.0, np.float32)
    ref_ops.exit_projection(rows, None, ref_tm.DEFAULT_EPS, positions, got_nogain)
    return {"gain": gain, "rows": rows, "positions": positions, "out": got,
            "out_nogain": got_nogain}


def gen_labels():
    out = {}
    for name, spec in LABEL_CASES.items():
        ckpts, final = make_label_inputs(spec)
        states = ref_cal.CollectedStates(checkpoint_states=ckpts, final_states=final,
                                         token_count=len(final), corpus_digest="golden")
        ds = ref_cal.compute_labels(states, spec["tau"])
        out[f"{name}__digest"] = np.frombuffer(
            digest(final, *[ckpts[k] for k in sorted(ckpts)]).encode(), np.uint8)
        for k in sorted(ckpts):
            out[f"{name}__sims_{k}"] = ds.similarities[k]
            out[f"{name}__labels_{k}"] = ds.labels[k]
        out[f"{name}__zero"] = np.array([ds.zero_norm_count])
    return out


def gen_posthoc():
    """Desk model (L=12, d=64), rigged + trained banks, synthetic captures
    (test_runtime.py:16-19 recipe) — exit maps and logits from the reference."""
    model = earlyexit.build_model(earlyexit.desk_config())
    out = {"final_norm": model.final_norm, "lm_head": model.lm_head}
    rigged = make_rigged_bank(model.config, hot_layers=(7,))
    corpus = earlyexit.load_corpus(earlyexit.fixtures.corpus_path())
    trained = ref_cal.calibrate(model, corpus[:300], ref_cal.CalibrationConfig(epochs=25, seed=11))
    for bname, bank in (("rigged", rigged), ("trained", trained)):
        out[f"{bname}__ckpts"] = np.array(bank.checkpoints, np.int64)
        out[f"{bname}__eps"] = np.array([bank.eps], np.float64)
        for k in bank.checkpoints:
            out[f"{bname}__wd_{k}"] = bank.routers[k].w_down
            out[f"{bname}__wu_{k}"] = bank.routers[k].w_up
    # check the in-repo rigged recipe restates the reference fixture exactly
    for k in rigged.checkpoints:
        wd, wu = rigged_router_arrays(64, hot=(k == 7), scale=64.0)
        assert np.array_equal(wd, rigged.routers[k].w_down)
        assert np.array_equal(wu, rigged.routers[k].w_up)
    cases = []
    for seed, n, zero_row in ((1234, 40, None), (1235, 6, (8, 2)), (1236, 300, None),
                              (1237, 1, None), (1238, 97, (4, 5))):
        states = posthoc_states(seed, n, zero_row)
        for bname, bank in (("rigged", rigged), ("trained", trained)):
            for theta in (1.0, 0.9, 0.85, 0.5, 0.1):
                for mode in (ref_rt.PER_TOKEN, ref_rt.BATCH_UNANIMOUS):
                    for k_min in (0, 8):
                        cfg = ref_rt.RuntimeConfig(exit_threshold=theta, mode=mode, k_min=k_min)
                        logits, exits = ref_rt.posthoc_select(model, states, bank, cfg)
                        key = f"c{len(cases)}"
                        cases.append((seed, n, zero_row, bname, theta, mode, k_min))
                        out[f"{key}__exits"] = exits
                        if n <= 40 and k_min == 0 and theta in (1.0, 0.5):
                            out[f"{key}__logits"] = logits
                        out[f"{key}__digest"] = np.frombuffer(digest(*states).encode(), np.uint8)
        # per-checkpoint scores for the trained bank (decode/all-checkpoint path)
        for k in trained.checkpoints:
            out[f"s{seed}__trained_scores_{k}"] = ref_ops.fused_layernorm_route(
                states[k + 1], trained.routers[k], eps=trained.eps)
    meta = np.array([repr(c) for c in cases])
    out["cases"] = meta
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "route.npz"), **gen_route())
    np.savez_compressed(os.path.join(HERE, "compact.npz"), **gen_compact())
    np.savez_compressed(os.path.join(HERE, "projection.npz"), **gen_projection())
    np.savez_compressed(os.path.join(HERE, "labels.npz"), **gen_labels())
    np.savez_compressed(os.path.join(HERE, "posthoc.npz"), **gen_posthoc())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
