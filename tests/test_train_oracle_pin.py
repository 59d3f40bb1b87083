"""Pins the training oracle (oracle/train_oracle.py + the Rng restatement in
oracle/ks_oracle.c) to the unmodified reference: committed fixtures made by
tests/golden/make_train_fixtures.py, plus live comparisons against
oracle/_ref/libkernelseer_ref.so when it is present."""
import os
import tempfile

import numpy as np
import pytest

from oracle import train_oracle as TO
from tests.golden.make_train_fixtures import (RNG_CASES, SHUFFLE_CASES, STEPS, TRAIN_MODELS, LR,
                                              with_dropout)
from tests.util import golden_path

GOLD = np.load(golden_path("train_golden.npz"))


def test_rng_streams_match_reference():
    import ctypes as C

    L = TO._okso()
    for seed, stream, n in RNG_CASES:
        u = np.zeros(n)
        L.kso_uniforms(seed, stream, n, u.ctypes.data_as(C.POINTER(C.c_double)))
        np.testing.assert_array_equal(u, GOLD[f"rng/{seed}/{stream}"])
    for seed, epoch, n in SHUFFLE_CASES:
        np.testing.assert_array_equal(TO.shuffle(seed, epoch, n), GOLD[f"shuffle/{seed}/{epoch}/{n}"])


def _ckpt(stem, drop, tmp):
    path = golden_path(stem + ".ckpt")
    return with_dropout(path, os.path.join(tmp, stem + "_drop.ckpt")) if drop else path


@pytest.mark.parametrize("drop", [False, True])
@pytest.mark.parametrize("stem", TRAIN_MODELS)
def test_loss_and_gradients_match_reference(stem, drop):
    """model_loss_gradients summed over a batch (models.cpp:788-797), fp64:
    the restatement agrees to rounding (1e-12 relative to the largest entry)."""
    key = f"{stem}/{'drop' if drop else 'nodrop'}"
    with tempfile.TemporaryDirectory() as tmp:
        ck = TO.Checkpoint(_ckpt(stem, drop, tmp))
    tok, tgt, idx = GOLD[key + "/tok"], GOLD[key + "/tgt"], GOLD[key + "/idx"]
    masks = TO.dropout_masks(ck, 11, 2, idx) if drop else None
    assert (masks is None) == (not drop)
    loss, G, _ = TO.loss_and_grads(ck, ck.tensors, tok, tgt, masks)
    ref = GOLD[key + "/grads"]
    assert abs(loss - float(GOLD[key + "/loss"])) <= 1e-12 * abs(loss)
    assert np.abs(ck.flat(G) - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("drop", [False, True])
@pytest.mark.parametrize("stem", TRAIN_MODELS)
def test_optimizer_steps_match_reference(stem, drop):
    """train_model's batch body (/ batch, clip 5.0, Adam) for 3 steps."""
    key = f"{stem}/{'drop' if drop else 'nodrop'}"
    with tempfile.TemporaryDirectory() as tmp:
        ck = TO.Checkpoint(_ckpt(stem, drop, tmp))
    tok, tgt, idx = GOLD[key + "/tok"], GOLD[key + "/tgt"], GOLD[key + "/idx"]
    flat = ck.flat()
    adam = TO.Adam(lr=LR)
    for s in range(STEPS):
        masks = TO.dropout_masks(ck, 11, 1 + s, idx) if drop else None
        flat, loss = TO.train_step(ck, flat, adam, tok, tgt, 5.0, masks)
        ref = GOLD[key + "/train_params"][s]
        assert abs(loss - GOLD[key + "/train_loss"][s]) <= 1e-12 * abs(loss)
        np.testing.assert_allclose(flat, ref, rtol=0, atol=1e-12)


def test_live_reference_small_model():
    """The trained small attn model (72k parameters) against the live reference."""
    from oracle.oracle import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libkernelseer_ref.so not built")
    from tests.golden.make_train_fixtures import ref_lib, ref_loss_grads

    path = golden_path("attn_small_trained.ckpt")
    ck = TO.Checkpoint(path)
    rng = np.random.default_rng(3)
    B = 24
    tok = np.stack([rng.integers(0, len(ck.inputs[f]), B) for f in range(7)], 1).astype(np.int32)
    tgt = np.stack([rng.integers(0, v, B) for v in ck.vsizes], 1).astype(np.int32)
    loss_r, g_r = ref_loss_grads(ref_lib(), path, tok, tgt)
    loss, G, _ = TO.loss_and_grads(ck, ck.tensors, tok, tgt)
    assert abs(loss - loss_r) <= 1e-12 * loss
    assert np.abs(ck.flat(G) - g_r).max() <= 1e-12 * np.abs(g_r).max()
