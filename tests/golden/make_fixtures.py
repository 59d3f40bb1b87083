"""Generates the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/make_fixtures.py            # small committed fixtures
    python tests/golden/make_fixtures.py --big      # + the default-size (tracked)
                                                    #   trained checkpoint (~2 min, 8 cores)

Checkpoints are written by the reference's own init_model/train +
save_checkpoint (compiled from /root/reference/proj/src and
/root/reference/proj/bindings/module.cpp by oracle/Makefile), and the
expected beams in golden.npz are the reference's own beam_search /
constrained_beam_search / greedy_decode outputs.  tests/test_oracle_pin.py
checks the C restatement (oracle/ks_oracle.c) against them bit for bit.
"""
from __future__ import annotations

import argparse
import itertools
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import RefModel, ref_init_save_spec, REF_DIR  # noqa: E402

# tiny_spec(arity, sizes) of proj/tests/test_util.hpp:50-60 as spec lines
TINY = {
    "s3423": "TinyKernel|p0=0-2|p1=0-3|p2=0-1|p3=0-2",
    "s222": "TinyKernel|p0=0-1|p1=0-1|p2=0-1",
    "s434": "TinyKernel|p0=0-3|p1=0-2|p2=0-3",
    "s232": "TinyKernel|p0=0-1|p1=0-2|p2=0-1",
    "s22": "TinyKernel|p0=0-1|p1=0-1",
}
TINY_MODELS = [  # (file stem, variant, spec key, seed)
    ("tiny_attn_s3423", "attn", "s3423", 11),
    ("tiny_attn2_s3423", "attn-2", "s3423", 11),
    ("tiny_encdec_s3423", "enc-dec", "s3423", 11),
    ("tiny_attn_s222", "attn", "s222", 3),
    ("tiny_encdec_s222", "enc-dec", "s222", 4),
    ("tiny_attn_s434", "attn", "s434", 23),
    ("tiny_attn_s232", "attn", "s232", 5),
    ("tiny_attn_s22", "attn", "s22", 29),
    ("tiny_hybrid2_s3423", "hybrid-2", "s3423", 11),
    ("tiny_hybrid_s3423", "hybrid", "s3423", 12),
    ("tiny_hybrid2_s434", "hybrid-2", "s434", 23),
]

BUDGET_LINE = "budget tiny_budget {b} p0=0.5,p1=1.0,p2=1.5"


def tiny_inputs():
    # tiny_vocab: every input field holds {1, 2} -> token ids {0, 1}
    return np.array(list(itertools.product([0, 1], repeat=7))[::9], np.int32)


def write_specs(ks):
    """builtin_specs() and search_space_size() as the reference reports them."""
    import json

    specs = [{"name": s.name, "params": [[n, list(v)] for n, v in s.params],
              "search_space": ks.search_space_size(s)} for s in ks.builtin_specs()]
    with open(os.path.join(HERE, "builtin_specs.json"), "w") as f:
        json.dump(specs, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--specs-only", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, REF_DIR)
    import _kernelseer as ks  # the reference's own pybind module

    write_specs(ks)
    if args.specs_only:
        return

    golden = {}
    for stem, variant, skey, seed in TINY_MODELS:
        path = os.path.join(HERE, stem + ".ckpt")
        ref_init_save_spec(path, variant, TINY[skey], seed)
        rm = RefModel(path)
        tok = tiny_inputs()
        golden[f"{stem}/tok"] = tok
        golden[f"{stem}/greedy"] = rm.greedy(tok)
        for k in (1, 2, 3, 8, 64):
            r = rm.beam(tok, k)
            golden[f"{stem}/k{k}/tokens"] = r["tokens"]
            golden[f"{stem}/k{k}/log_prob"] = r["log_prob"]
            golden[f"{stem}/k{k}/count"] = r["count"]
        for b in (1.0, 2.5):
            r = rm.beam(tok, 4, preds_text="membership\n" + BUDGET_LINE.format(b=b))
            for key in ("tokens", "log_prob", "count", "status", "fail_step"):
                golden[f"{stem}/budget{b}/{key}"] = r[key]
            golden[f"{stem}/budget{b}/fail_name"] = np.array(r["fail_name"])

    # small trained attn model on the ConvAsm1x1U synthetic task (committed)
    spec = ks.builtin_spec("ConvAsm1x1U")
    ds = ks.generate_synthetic(spec, 5000, seed=7, difficulty="moderate")
    train, test = ks.split(ds, 0.2, seed=7)
    cfg = ks.ModelConfig(variant="attn", pre_attention_size=32, post_attention_size=64,
                         dropout=0.0, recurrent_dropout=0.0)
    params, log = ks.train(cfg, spec, train.samples[:2000], test.samples[:200], epochs=6,
                           batch_size=32, seed=1, threads=8, learning_rate=3e-3)
    small = os.path.join(HERE, "attn_small_trained.ckpt")
    ks.save_checkpoint(params, small)
    print("small model test acc", log[-1]["test_avg_acc"])
    rm = RefModel(small)
    desc = np.array([[s.descriptor[f] for f in "nchwkyx"] for s in test.samples[:96]], np.int64)
    tok, bad = rm.encode(desc)
    assert bad == 0
    golden["small/desc"] = desc
    golden["small/tok"] = tok
    golden["small/greedy"] = rm.greedy(tok)
    names = [p for p, _ in spec.params]
    for k in (1, 5):
        r = rm.beam(tok, k)
        golden[f"small/k{k}/tokens"] = r["tokens"]
        golden[f"small/k{k}/log_prob"] = r["log_prob"]
    line = "membership\nbudget bud 28 " + ",".join(f"{n}=1.0" for n in names)
    r = rm.beam(tok, 5, desc, preds_text=line)
    for key in ("tokens", "log_prob", "count", "status", "fail_step"):
        golden[f"small/constrained/{key}"] = r[key]
    # small trained hybrid-2 (the reference's default variant) on the same task
    cfg = ks.ModelConfig(variant="hybrid-2", conv_layers=[(16, 3, 1), (8, 3, 1)], decoder_cell_size=32,
                         dropout=0.0, recurrent_dropout=0.0)
    params, log = ks.train(cfg, spec, train.samples[:2000], test.samples[:200], epochs=6,
                           batch_size=32, seed=1, threads=8, learning_rate=3e-3)
    hyb = os.path.join(HERE, "hybrid2_small_trained.ckpt")
    ks.save_checkpoint(params, hyb)
    print("small hybrid-2 test acc", log[-1]["test_avg_acc"])
    rm = RefModel(hyb)
    golden["hyb/greedy"] = rm.greedy(tok)
    for k in (1, 5):
        r = rm.beam(tok, k)
        golden[f"hyb/k{k}/tokens"] = r["tokens"]
        golden[f"hyb/k{k}/log_prob"] = r["log_prob"]
    r = rm.beam(tok, 5, desc, preds_text=line)
    for key in ("tokens", "log_prob", "count", "status", "fail_step"):
        golden[f"hyb/constrained/{key}"] = r[key]
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **golden)
    print("wrote", len(golden), "arrays")

    if args.big:
        cfg = ks.ModelConfig(variant="attn", dropout=0.0, recurrent_dropout=0.0)
        params, log = ks.train(cfg, spec, train.samples[:2000], test.samples[:200], epochs=4,
                               batch_size=32, seed=1, threads=8, learning_rate=2e-3)
        ks.save_checkpoint(params, os.path.join(HERE, "attn_default_trained.ckpt"))
        print("default model test acc", log[-1]["test_avg_acc"])


if __name__ == "__main__":
    main()
