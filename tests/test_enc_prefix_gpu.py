"""Shared-prefix encoder (ks_engine.cu encode_prefix / enc_prefix_gather): encoder
steps run once per token prefix (fan-out epilogue over the previous step's
prefixes) and gathered per config must give decodes bit-identical to running every
encoder step per config (KS_ENC_PREFIX=0) -- on the BASELINE model at chunk sizes
that cover different step counts (all 7 steps of both directions at 60,000 configs)
and on random models."""
import os

import numpy as np
import pytest

from tests.util import have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a GPU")]


def _decode(path, prec, tok, k, preds, table, chunk=None):
    from paper_2404_10162_b200._cabi import Engine

    # KS_ENC_PREFIX_MIN=0: the prefix steps also at the small chunks of these cases
    env = {"KS_ENC_PREFIX": "1" if table else "0", "KS_ENC_PREFIX_MIN": "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        e = Engine(path, 0, prec)
    finally:
        for name, val in old.items():
            if val is None:
                os.environ.pop(name)
            else:
                os.environ[name] = val
    if chunk:
        e.set_chunk(chunk)
    return e.beam(tok, k, None, preds)


def _same(a, b):
    for key in ("tokens", "log_prob", "count", "status"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("prec,B,chunk", [("f16x3", 6000, 2500), ("bf16", 6000, 2500), ("f16x3", 60000, None),
                                          ("f16x3", 3000, 700)])
def test_tables_bit_identical_default_model(prec, B, chunk):
    from paper_2404_10162_b200 import workloads as W
    from paper_2404_10162_b200._cabi import Engine

    path = W.DEFAULT_CKPT
    e = Engine(path, 0, prec)
    tok = e.encode(e.synthetic(B, W.SEED, 123))
    preds = W.predicate_dicts(path)
    _same(_decode(path, prec, tok, 5, preds, True, chunk), _decode(path, prec, tok, 5, preds, False, chunk))


@pytest.mark.parametrize("case", range(3))
def test_tables_bit_identical_random_models(case, tmp_path):
    import paper_2404_10162_b200 as ks
    from oracle.oracle import OracleModel
    from tests.test_fuzz_gpu import _model

    variant, n_a, spec = [("attn", 64, "ConvAsm1x1U"), ("attn-2", 128, "ConvOclDirectFwd1x1"),
                          ("attn", 192, "ConvAsmBwdWrW3x3")][case]
    path = _model(ks, variant, n_a, 128, 2, spec, 300 + case, str(tmp_path / "m.ckpt"))
    o = OracleModel(path)
    rng = np.random.default_rng(case)
    B = 700
    tok = np.stack([rng.integers(0, len(o.input_values[f]), B) for f in range(7)], 1).astype(np.int32)
    preds = [o.membership()]
    _same(_decode(path, "f16x3", tok, 4, preds, True), _decode(path, "f16x3", tok, 4, preds, False))
