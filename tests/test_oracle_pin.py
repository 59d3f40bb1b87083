"""Pins the CPU oracle (oracle/ks_oracle.c) to the reference.

* against golden.npz, produced by the reference's own beam_search /
  constrained_beam_search / greedy_decode (tests/golden/make_fixtures.py):
  bit-exact tokens AND fp64 log-probs;
* against the live reference build (oracle/_ref/libkernelseer_ref.so, compiled
  from /root/reference/proj/src) on random configs when it is present.
"""
import os

import numpy as np
import pytest

from tests.util import BIG_CKPT, golden_path
from oracle.oracle import OracleModel, RefModel, ref_available
from tests.golden.make_fixtures import TINY_MODELS

TINY_STEMS = [m[0] for m in TINY_MODELS]


def _budget_pred(o, b):
    return o.budget({"p0": 0.5, "p1": 1.0, "p2": 1.5}, b)


@pytest.mark.parametrize("stem", TINY_STEMS)
def test_oracle_matches_reference_golden_tiny(golden, stem):
    o = OracleModel(golden_path(stem + ".ckpt"))
    tok = golden[f"{stem}/tok"]
    assert (o.greedy(tok) == golden[f"{stem}/greedy"]).all()
    for k in (1, 2, 3, 8, 64):
        r = o.beam(tok, k)
        np.testing.assert_array_equal(r["count"], golden[f"{stem}/k{k}/count"])
        np.testing.assert_array_equal(r["tokens"], golden[f"{stem}/k{k}/tokens"])
        # bit-identical fp64 log-probs (same operation order, no FMA)
        np.testing.assert_array_equal(r["log_prob"], golden[f"{stem}/k{k}/log_prob"])
    for b in (1.0, 2.5):
        r = o.beam(tok, 4, preds=[o.membership(), _budget_pred(o, b)])
        g = f"{stem}/budget{b}"
        np.testing.assert_array_equal(r["status"], golden[g + "/status"])
        np.testing.assert_array_equal(r["tokens"], golden[g + "/tokens"])
        np.testing.assert_array_equal(r["log_prob"], golden[g + "/log_prob"])
        ex = r["status"] == 1
        np.testing.assert_array_equal(r["fail_step"][ex], golden[g + "/fail_step"][ex])
        names = np.array(["membership:TinyKernel", "tiny_budget"])
        assert (names[r["fail_pred"][ex]] == golden[g + "/fail_name"][ex]).all()


def test_oracle_matches_reference_golden_trained(golden):
    o = OracleModel(golden_path("attn_small_trained.ckpt"))
    tok, desc = golden["small/tok"], golden["small/desc"]
    t2, bad = o.encode_problem(desc)
    assert (bad == -1).all() and (t2 == tok).all()
    assert (o.greedy(tok) == golden["small/greedy"]).all()
    for k in (1, 5):
        r = o.beam(tok, k)
        np.testing.assert_array_equal(r["tokens"], golden[f"small/k{k}/tokens"])
        np.testing.assert_array_equal(r["log_prob"], golden[f"small/k{k}/log_prob"])
    r = o.beam(tok, 5, desc, preds=[o.membership(), o.budget({n: 1.0 for n in o.names}, 28)])
    np.testing.assert_array_equal(r["status"], golden["small/constrained/status"])
    np.testing.assert_array_equal(r["tokens"], golden["small/constrained/tokens"])
    np.testing.assert_array_equal(r["log_prob"], golden["small/constrained/log_prob"])


def test_tie_order_known_answer():
    """decoding_test.cpp:159-174: zeroed heads -> every sequence ties; order
    {0,0,0},{0,0,1},{0,1,0},{0,1,1},{0,2,0}."""
    import tempfile

    from tests import ckpt_util

    with tempfile.TemporaryDirectory() as tmp:
        path = ckpt_util.modified(golden_path("tiny_attn_s232.ckpt"), os.path.join(tmp, "z.ckpt"),
                                  lambda t: [t[n].fill(0) for n in t if n.startswith("head.")])
        o = OracleModel(path)
        r = o.beam(np.array([[0, 1, 0, 1, 0, 1, 0]]), 5)
        assert r["tokens"][0].tolist() == [[0, 0, 0], [0, 0, 1], [0, 1, 0], [0, 1, 1], [0, 2, 0]]
        assert r["min_gap"][0] == 0.0  # flagged tie-adjacent


@pytest.mark.skipif(not ref_available(), reason="reference build absent")
def test_oracle_matches_live_reference_random():
    o = OracleModel(golden_path("attn_small_trained.ckpt"))
    r = RefModel(golden_path("attn_small_trained.ckpt"))
    rng = np.random.default_rng(5)
    tok = np.stack([rng.integers(0, len(o.input_values[f]), 64) for f in range(7)], 1).astype(np.int32)
    a, b = o.beam(tok, 7), r.beam(tok, 7)
    np.testing.assert_array_equal(a["tokens"], b["tokens"])
    np.testing.assert_array_equal(a["log_prob"], b["log_prob"])


@pytest.mark.skipif(not ref_available(),
                    reason="reference build or default-size checkpoint absent")
def test_oracle_matches_live_reference_default_size():
    o, r = OracleModel(BIG_CKPT), RefModel(BIG_CKPT)
    rng = np.random.default_rng(6)
    tok = np.stack([rng.integers(0, len(o.input_values[f]), 8) for f in range(7)], 1).astype(np.int32)
    a, b = o.beam(tok, 5, threads=8), r.beam(tok, 5, threads=8)
    np.testing.assert_array_equal(a["tokens"], b["tokens"])
    np.testing.assert_array_equal(a["log_prob"], b["log_prob"])


def test_oracle_matches_reference_golden_trained_hybrid2(golden):
    """The reference's default variant (hybrid-2): conv stack + seeded bi-LSTMs
    (models.cpp:296-371), beam over static distributions."""
    o = OracleModel(golden_path("hybrid2_small_trained.ckpt"))
    tok, desc = golden["small/tok"], golden["small/desc"]
    assert (o.greedy(tok) == golden["hyb/greedy"]).all()
    for k in (1, 5):
        r = o.beam(tok, k)
        np.testing.assert_array_equal(r["tokens"], golden[f"hyb/k{k}/tokens"])
        np.testing.assert_array_equal(r["log_prob"], golden[f"hyb/k{k}/log_prob"])
    r = o.beam(tok, 5, desc, preds=[o.membership(), o.budget({n: 1.0 for n in o.names}, 28)])
    np.testing.assert_array_equal(r["status"], golden["hyb/constrained/status"])
    np.testing.assert_array_equal(r["tokens"], golden["hyb/constrained/tokens"])
    np.testing.assert_array_equal(r["log_prob"], golden["hyb/constrained/log_prob"])
