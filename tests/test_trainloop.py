"""The drop-in `train` API (reference bindings/module.cpp:222-256 ->
train_model, models.cpp:862-969) against the reference's own runs
(tests/golden/make_trainloop_fixtures.py): init_model must be bit-identical
(same Rng draws, fp32-rounded like a checkpoint), and two epochs of training
with dropout 0.2 / 0.2 must follow the reference trajectory (same shuffles,
same per-sample dropout masks; fp32 GPU arithmetic vs the reference's fp64)."""
import json
import os
import tempfile

import numpy as np
import pytest

from tests import ckpt_util
from tests.golden.make_trainloop_fixtures import CONFIG, INIT_N, TRAIN
from tests.util import golden_path, have_gpu


def _data(ks):
    with open(golden_path("trainloop_data.json")) as f:
        d = json.load(f)
    mk = lambda rows: [ks.Sample(r["descriptor"], r["params"], d["kernel"], "fp32") for r in rows]
    return ks.builtin_spec(d["kernel"]), mk(d["train"]), mk(d["test"])


def test_init_model_matches_reference_bit_for_bit():
    import paper_2404_10162_b200 as ks

    spec, train, test = _data(ks)
    params = ks.init_model(ks.ModelConfig(**CONFIG), spec, train[:INIT_N[0]] + test[:INIT_N[1]], seed=TRAIN["seed"])
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "init.ckpt")
        ks.save_checkpoint(params, path)
        h_ours, order_ours, t_ours = ckpt_util.read(path)
        assert open(path, "rb").read() == open(golden_path("trainloop_init.ckpt"), "rb").read()
    h_ref, order_ref, t_ref = ckpt_util.read(golden_path("trainloop_init.ckpt"))
    assert h_ours == h_ref and order_ours == order_ref


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs a GPU")
def test_train_follows_reference_trajectory():
    import paper_2404_10162_b200 as ks

    spec, train, test = _data(ks)
    params, log = ks.train(ks.ModelConfig(**CONFIG), spec, train, test, **TRAIN)
    with open(golden_path("trainloop_log.json")) as f:
        ref_log = json.load(f)
    for ours, ref in zip(log, ref_log):
        assert ours["epoch"] == ref["epoch"]
        for key in ("train_loss", "test_loss"):
            assert abs(ours[key] - ref[key]) <= 2e-3 * abs(ref[key]), (key, ours, ref)
        for key in ("train_avg_acc", "test_avg_acc"):
            assert abs(ours[key] - ref[key]) <= 1.0, (key, ours, ref)  # percent
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "ours.ckpt")
        ks.save_checkpoint(params, path)
        _, order, ours = ckpt_util.read(path)
    _, order_ref, ref = ckpt_util.read(golden_path("trainloop_ref.ckpt"))
    assert order == order_ref
    steps = TRAIN["epochs"] * -(-len(train) // TRAIN["batch_size"])
    for name in order:
        a, b = ours[name].astype(np.float64), ref[name].astype(np.float64)
        if name == "attn.out.bias":
            # shift-invariant under the softmax: its gradient is exactly 0, so Adam only
            # normalises rounding noise (fp64 ~1e-18 -> eps-damped; fp32 ~1e-8 -> up to lr
            # per step); it never changes the model's output
            assert np.abs(a - b).max() <= TRAIN["learning_rate"] * steps
            continue
        rel = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-12)
        assert rel <= 2e-3, f"{name}: relative L2 difference {rel:.2e}"
    # the trained model decodes through the engine
    beams = ks.predict(params, train[0].descriptor, beam_width=3)
    assert len(beams) == 3
