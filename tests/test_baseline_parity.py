"""GPU parity at the BASELINE.json workloads, against the REFERENCE's own
decodes (tests/golden/baseline_parity.npz, made by
tests/golden/make_baseline_fixtures.py with the unmodified reference; the fp64
oracle's tie flags beside them).

* cfg2: the timed 4,096-config prefix of the 65,536-config workload plus a
  random 4,096 of the rest, beam 5, membership +
  budget 60, the default-size trained model.
* cfg1: greedy decode of the 1,000-config workload, default-size model.
* cfg5: n_a = n_s = 1024, ConvAsmBwdWrW1x1, beam 16, membership + budget 40;
  the checkpoint is rebuilt here by our init_model and must hash to the
  reference-written file the fixtures were decoded on.

Bar: identical token sequences, rank order, counts and
exhaustion on every config the oracle does not flag tie-adjacent; log-probs
within 1e-4 relative.  The BF16 path is reduced precision: its agreement is
measured and must stay above a floor.
"""
import os

import numpy as np
import pytest

from paper_2404_10162_b200 import workloads as W
from tests.util import ROOT, TIE_REL, compare_beams, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a GPU")]

FX = os.path.join(ROOT, "tests", "golden", "baseline_parity.npz")


@pytest.fixture(scope="module")
def fx():
    return dict(np.load(FX))


def ref_dict(fx, cfg):
    out = {k.split("/", 1)[1]: v for k, v in fx.items() if k.startswith(cfg + "/")}
    return out


def engine(path, precision):
    from paper_2404_10162_b200._cabi import Engine
    return Engine(path, 0, precision)


def agreement(g, ref):
    top1 = (g["tokens"][:, 0] == ref["tokens"][:, 0]).all(axis=1)
    full = (g["tokens"] == ref["tokens"]).all(axis=(1, 2))
    return float(top1.mean()), float(full.mean())


@pytest.mark.parametrize("precision", ["f16x3", "fp32"])
def test_cfg2_prefix_and_random_sample(fx, precision):
    r = ref_dict(fx, "cfg2")
    e = engine(W.DEFAULT_CKPT, precision)
    g = e.beam(r["tok"], 5, r["desc"], W.predicate_dicts(W.DEFAULT_CKPT))
    n, ties, bad = compare_beams(g, r)
    assert len(r["tok"]) == 8192 and n >= 0.95 * 8192, (n, ties)
    assert not bad, f"{len(bad)} mismatching of {n} compared ({ties} tie-adjacent); first {bad[:8]}"


def test_cfg2_bf16_agreement(fx):
    """Reduced precision: decoded-sequence agreement with the reference on the
    8,192 configs (reported by bench.py as `agreement`); a floor guards
    against regressions, not a parity claim."""
    r = ref_dict(fx, "cfg2")
    g = engine(W.DEFAULT_CKPT, "bf16").beam(r["tok"], 5, r["desc"], W.predicate_dicts(W.DEFAULT_CKPT))
    top1, full = agreement(g, r)
    print(f"bf16 agreement vs reference: top-1 {top1:.4f}, full list {full:.4f}")
    assert top1 >= 0.97 and full >= 0.85


@pytest.mark.parametrize("precision", ["f16x3", "fp32"])
def test_cfg1_greedy_1000(fx, precision):
    r = ref_dict(fx, "cfg1")
    g = engine(W.DEFAULT_CKPT, precision).greedy(r["tok"])
    tie = r["min_gap"] < TIE_REL
    bad = np.nonzero(~tie & ~(g == r["tokens"]).all(axis=1))[0]
    assert len(r["tok"]) == 1000 and tie.mean() < 0.05
    assert not len(bad), f"{len(bad)} mismatching greedy decodes; first {bad[:8]}"


@pytest.mark.parametrize("precision", ["f16x3", "fp32"])
def test_cfg5_large_model_beam16(fx, precision):
    r = ref_dict(fx, "cfg5")
    path = W.cfg5_checkpoint_ours()
    assert W.sha256(path) == str(r["sha256"]), "cfg5 checkpoint differs from the reference-written one"
    g = engine(path, precision).beam(r["tok"], 16, r["desc"], W.predicate_dicts(path))
    n, ties, bad = compare_beams(g, r)
    # beam 16 over 10 positions: ~13% of these untrained-but-peaked configs have a
    # deciding gap under 1e-4 relative in fp64 and are excluded by the tie rule
    assert n >= 0.8 * len(r["tok"]), (n, ties)
    assert not bad, f"{len(bad)} mismatching of {n} compared ({ties} tie-adjacent); first {bad[:8]}"


def test_cfg2_chunked_and_sharded_equal_whole(fx):
    """The configs' results do not depend on how the batch is cut: small
    chunks, and contiguous shards decoded separately (the multi-GPU split),
    give the decodes of one call (up to tie-adjacent reorderings)."""
    r = ref_dict(fx, "cfg2")
    tok, desc = r["tok"][:2048], r["desc"][:2048]
    preds = W.predicate_dicts(W.DEFAULT_CKPT)
    e = engine(W.DEFAULT_CKPT, "f16x3")
    whole = e.beam(tok, 5, desc, preds)
    parts = [e.beam(tok[lo:lo + 512], 5, desc[lo:lo + 512], preds) for lo in range(0, 2048, 512)]
    e.set_chunk(300)
    chunked = e.beam(tok, 5, desc, preds)
    sub = {k: v[:2048] for k, v in r.items() if k in ("tokens", "log_prob", "count", "status", "fail_pred",
                                                      "fail_step", "min_gap")}
    for g in (whole, chunked, {k: np.concatenate([p[k] for p in parts]) for k in whole}):
        n, ties, bad = compare_beams(g, sub)
        assert not bad
