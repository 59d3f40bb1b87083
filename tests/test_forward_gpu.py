"""model_forward, the SequencePredictor stepping facade and the beam
rescoring oracle on the GPU (ks_forward_batch), against the fp64 oracle.

Reference behaviour pinned:
* model_forward with / without teacher tokens (models.cpp:495-514): per
  position distributions; the teacher's tokens are fed back, else the argmax.
* teacher forcing with the greedy tokens == the free run (models_test.cpp:319-335).
* every returned beam rescored by the teacher-forced scorer matches its
  log-prob (decoding_test.cpp:36-66, 223-272; acceptance_test.cpp:184-212):
  here within 1e-4 relative of the fp64 score, and the GPU scorer agrees with
  the GPU beam lp to fp32 rounding.
* step(): StateError past the end, IndexError for an out-of-range fed token.
"""
import math
import os

import numpy as np
import pytest

from oracle.oracle import OracleModel
from paper_2404_10162_b200 import workloads as W
from tests.golden.make_fixtures import TINY_MODELS
from tests.util import ROOT, TIE_REL, compare_beams, golden_path, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a GPU")]

MODELS = ["attn_small_trained", "hybrid2_small_trained"] + [m[0] for m in TINY_MODELS]


def engine(path, precision="f16x3"):
    from paper_2404_10162_b200._cabi import Engine
    return Engine(path, 0, precision)


def tokens(o, B, seed):
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, len(o.input_values[f]), B) for f in range(7)], 1).astype(np.int32)


@pytest.mark.parametrize("precision", ["f16x3", "fp32"])
@pytest.mark.parametrize("stem", MODELS)
def test_model_forward_teacher_forced(stem, precision):
    path = golden_path(stem + ".ckpt")
    o, e = OracleModel(path), engine(path, precision)
    tok = tokens(o, 64, 3)
    rng = np.random.default_rng(4)
    teach = np.stack([rng.integers(0, v, len(tok)) for v in o.vsizes], 1).astype(np.int32)
    dists, fed, score = e.forward(tok, teach)
    assert (fed == teach).all()
    for b in range(len(tok)):
        ref = o.forward(tok[b], teach[b])
        for p in range(o.T):
            np.testing.assert_allclose(dists[p][b], ref[p], rtol=0, atol=2e-5)
        s = o.score(tok[b], list(teach[b]))
        assert abs(score[b] - s) <= 1e-4 * max(1.0, abs(s))


@pytest.mark.parametrize("stem", MODELS)
def test_model_forward_free_run_equals_greedy(stem):
    """No teacher: the argmax is fed back -- the same tokens as greedy_decode,
    and teacher forcing with those tokens reproduces the free run
    (models_test.cpp:319-335)."""
    path = golden_path(stem + ".ckpt")
    o, e = OracleModel(path), engine(path)
    tok = tokens(o, 128, 5)
    d0, fed, s0 = e.forward(tok)
    assert (fed == e.greedy(tok)).all()
    d1, fed1, s1 = e.forward(tok, fed)
    assert (fed1 == fed).all()
    for p in range(o.T):
        np.testing.assert_array_equal(d0[p], d1[p])
    np.testing.assert_array_equal(s0, s1)
    # against the oracle's free run where its argmax is not a near tie
    a = o.beam(tok, 1, threads=8)
    ok = a["min_gap"] >= TIE_REL
    assert (fed[ok] == a["tokens"][ok, 0]).all()


def test_rescoring_default_model_beams():
    """decoding_test.cpp:38-46 / acceptance_test.cpp:224-299 on the default
    model: every GPU beam (membership + budget, beam 5) rescored by the fp64
    teacher-forced scorer matches its log-prob within 1e-4 relative, and by
    the GPU scorer (ks_forward_batch) within fp32 rounding."""
    fx = np.load(os.path.join(ROOT, "tests", "golden", "baseline_parity.npz"))
    tok, desc = fx["cfg2/tok"][:256], fx["cfg2/desc"][:256]
    o, e = OracleModel(W.DEFAULT_CKPT), engine(W.DEFAULT_CKPT)
    g = e.beam(tok, 5, desc, W.predicate_dicts(W.DEFAULT_CKPT))
    rows, seqs, lps = [], [], []
    for b in range(len(tok)):
        for i in range(g["count"][b]):
            rows.append(b)
            seqs.append(g["tokens"][b, i])
            lps.append(g["log_prob"][b, i])
    rows, seqs, lps = np.array(rows), np.array(seqs, np.int32), np.array(lps)
    _, _, gs = e.forward(tok[rows], seqs)
    assert np.all(np.abs(gs - lps) <= 1e-5 * np.maximum(1.0, np.abs(lps)))
    for j in range(0, len(rows), 3):  # a third of them through the fp64 scorer
        s = o.score(tok[rows[j]], list(seqs[j]))
        assert abs(s - lps[j]) <= 1e-4 * max(1.0, abs(s)), (j, s, lps[j])


def test_python_sequence_predictor_step_and_errors():
    import paper_2404_10162_b200 as ks

    path = golden_path("attn_small_trained.ckpt")
    params = ks.load_checkpoint(path)
    o = OracleModel(path)
    sp = ks.SequencePredictor(params)
    tok = [int(t) for t in tokens(o, 1, 9)[0]]
    enc = sp.encode(tok)
    st = sp.initial_state(enc)
    prev, fed = -1, []
    for p in range(sp.num_positions()):
        d = np.array(sp.step(enc, st, prev))
        assert st.position == p + 1 and len(d) == sp.vocab_size(p)
        prev = int(np.argmax(d))
        fed.append(prev)
    ref = o.forward(np.array(tok, np.int32), np.array(fed, np.int32))
    np.testing.assert_allclose(d, ref[-1], atol=2e-5)
    with pytest.raises(ks.KernelseerError, match="past the last output position"):
        sp.step(enc, st, 0)
    st2 = sp.initial_state(enc)
    sp.step(enc, st2, -1)
    with pytest.raises(ks.KernelseerError, match="out of range"):
        sp.step(enc, st2, 99)
    # batched model_forward through the Python API equals the stepping
    dists, scores = ks.model_forward(params, [tok], [fed])
    np.testing.assert_allclose(dists[0][-1], d, atol=0)
    assert math.isfinite(scores[0])


def test_engine_encode_oov_and_snap():
    """ks_encode_problems: OOV -> ValidationError naming the field and the row;
    allow_nearest snaps (encoding_test.cpp:132-146)."""
    from paper_2404_10162_b200._cabi import KsError

    e = engine(W.DEFAULT_CKPT)
    desc = np.array([[64, 16, 7, 7, 16, 1, 1], [3, 16, 7, 7, 16, 1, 1]], np.int64)
    with pytest.raises(KsError) as ex:
        e.encode(desc)
    assert ex.value.code == 5 and ex.value.field == "n" and "nearest" in str(ex.value)
    assert e.encode(desc, allow_nearest=True)[1].tolist() == [1, 0, 0, 0, 0, 0, 0]


def test_engine_group_preserves_config_order():
    """Two engines sharing one GPU (the multi-GPU sharding path, ks_group_*):
    contiguous shards, results in config order, identical to one engine."""
    from paper_2404_10162_b200._cabi import EngineGroup

    fx = np.load(os.path.join(ROOT, "tests", "golden", "baseline_parity.npz"))
    tok, desc = fx["cfg2/tok"][:1001], fx["cfg2/desc"][:1001]
    preds = W.predicate_dicts(W.DEFAULT_CKPT)
    one = engine(W.DEFAULT_CKPT).beam(tok, 5, desc, preds)
    ref = {k: fx["cfg2/" + k][:1001] for k in ("tokens", "log_prob", "count", "status", "fail_pred", "fail_step",
                                                "min_gap")}
    clear = ref["min_gap"] >= TIE_REL
    for devs in ([0, 0], [0, 0, 0]):
        grp = EngineGroup(W.DEFAULT_CKPT, devs)
        assert grp.size == len(devs)
        g = grp.beam(tok, 5, desc, preds)
        n, ties, bad = compare_beams(g, ref)
        assert not bad
        # shards hold the configs of one call, in order: same decodes as one engine
        np.testing.assert_array_equal(g["tokens"][clear], one["tokens"][clear])
        np.testing.assert_array_equal(g["count"], one["count"])
        np.testing.assert_allclose(g["log_prob"][clear], one["log_prob"][clear], rtol=1e-5)


def test_python_api_uses_every_visible_gpu():
    """ks.predict_batch / topk_metrics run on an engine group over all visible
    GPUs by default; an explicit device list (one GPU twice) gives the same
    beams as a single engine."""
    import paper_2404_10162_b200 as ks

    params = ks.load_checkpoint(W.DEFAULT_CKPT)
    assert params.num_devices == ks.device_count() >= 1
    fx = np.load(os.path.join(ROOT, "tests", "golden", "baseline_parity.npz"))
    names = ["n", "c", "h", "w", "k", "y", "x"]
    ds = [{n: int(v) for n, v in zip(names, row)} for row in fx["cfg2/desc"][:300]]
    preds = [ks.membership_predicate(params.spec),
             ks.resource_budget_predicate({n: 1.0 for n, _ in params.spec.params}, 60.0)]
    a = ks.predict_batch(params, ds, beam_width=5, predicates=preds)
    params.set_engine([0, 0])
    assert params.num_devices == 2
    b = ks.predict_batch(params, ds, beam_width=5, predicates=preds)
    def beams(res):  # a beam list per config, or its exhaustion record
        return [r if isinstance(r, dict) else [x["params"] for x in r] for r in res]

    assert any(isinstance(r, list) for r in a)
    assert beams(a) == beams(b)
