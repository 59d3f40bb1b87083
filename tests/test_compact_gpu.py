"""Parent compaction at the alpha-block positions (ks_engine.cu cp_count / cp_fill,
ks_gemm_tc.cu epilogue_compact): attention and the gate GEMM on each config's
distinct live parents, the epilogue writing their children.  The decodes are
checked against the REFERENCE's decodes (tests/golden/baseline_parity.npz) with
compaction on (the default) and off, and with position 1 compacted too
(KS_COMPACT_POS1=1), and against the fp64 oracle on random models (small
chunks, exhaustion, beam widths 2..16)."""
import os

import numpy as np
import pytest

from paper_2404_10162_b200 import workloads as W
from tests.util import ROOT, compare_beams, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a GPU")]

FX = os.path.join(ROOT, "tests", "golden", "baseline_parity.npz")


def _engine(path, prec, compact, pos1=False):
    from paper_2404_10162_b200._cabi import Engine

    env = {"KS_COMPACT": "1" if compact else "0", "KS_COMPACT_POS1": "1" if pos1 else "0"}
    old = {name: os.environ.get(name) for name in env}
    os.environ.update(env)
    try:
        return Engine(path, 0, prec)
    finally:
        for name, val in old.items():
            if val is None:
                os.environ.pop(name)
            else:
                os.environ[name] = val


def _ref(cfg):
    fx = np.load(FX)
    return {k.split("/", 1)[1]: fx[k] for k in fx.files if k.startswith(cfg + "/")}


@pytest.mark.parametrize("compact,pos1", [(True, False), (True, True), (False, False)])
@pytest.mark.parametrize("prec", ["f16x3", "bf16"])
def test_cfg2_fixtures(compact, pos1, prec):
    r = _ref("cfg2")
    e = _engine(W.DEFAULT_CKPT, prec, compact, pos1)
    g = e.beam(r["tok"], 5, r["desc"], W.predicate_dicts(W.DEFAULT_CKPT))
    if prec == "bf16":  # reduced precision: agreement floor only
        assert (g["tokens"][:, 0] == r["tokens"][:, 0]).all(axis=1).mean() >= 0.97
        return
    n, ties, bad = compare_beams(g, r)
    assert n >= 0.95 * len(r["tok"]), (n, ties)
    assert not bad, f"{len(bad)} mismatching of {n} compared ({ties} tie-adjacent); first {bad[:8]}"


@pytest.mark.parametrize("compact", [True, False])
def test_cfg5_fixtures(compact):
    r = _ref("cfg5")
    path = W.cfg5_checkpoint_ours()
    g = _engine(path, "f16x3", compact).beam(r["tok"], 16, r["desc"], W.predicate_dicts(path))
    n, ties, bad = compare_beams(g, r)
    assert n >= 0.8 * len(r["tok"]), (n, ties)
    assert not bad, f"{len(bad)} mismatching of {n} compared ({ties} tie-adjacent); first {bad[:8]}"


@pytest.mark.parametrize("case,pos1", [(0, False), (1, True), (3, False), (4, True), (7, False)])
def test_random_models_compacted(case, pos1, tmp_path):
    import paper_2404_10162_b200 as ks
    from oracle.oracle import OracleModel
    from tests.test_fuzz_gpu import CASES, _model

    variant, n_a, n_s, n_d, spec_name, k, B, prec = CASES[case]
    path = _model(ks, variant, n_a, n_s, n_d, spec_name, 100 + case, str(tmp_path / "m.ckpt"))
    o = OracleModel(path)
    rng = np.random.default_rng(case)
    tok = np.stack([rng.integers(0, len(o.input_values[f]), B) for f in range(7)], 1).astype(np.int32)
    budget = float(sum(np.median(v) for v in o.values))
    preds = [o.membership(), o.budget({nm: 1.0 for nm in o.names}, budget)]
    a = o.beam(tok, k, None, preds, threads=8)
    e = _engine(path, prec, True, pos1)
    e.set_chunk(97)
    g = e.beam(tok, k, None, preds)
    n, ties, bad = compare_beams(g, a)
    assert n >= 0.5 * B, (n, ties)
    assert not bad, f"{len(bad)} mismatching of {n} compared ({ties} tie-adjacent); first {bad[:6]}"
