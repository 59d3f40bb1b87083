"""Parity fixtures for the BASELINE.json workloads, made BY THE REFERENCE.

    python tests/golden/make_baseline_fixtures.py [cfg1|cfg2|cfg5 ...]   (~10 min on 8 cores)

Writes tests/golden/baseline_parity.npz:

* cfg2/*: 8,192 configs of BASELINE config 2 -- the timed 4,096-config prefix
  (configs 0..4095 of the 65,536) plus 4,096 drawn at random from the rest
   -- decoded by the unmodified reference's
  constrained_beam_search (oracle/_ref, beam 5, membership + budget 60) on the
  tracked default-size trained checkpoint.
* cfg1/*: BASELINE config 1, greedy_decode of configs 0..999.
* cfg5/*: 256 configs of BASELINE config 5 (n_a = n_s = 1024, ConvAsmBwdWrW1x1,
  beam 16, membership + budget 40) on the reference-written cfg5 checkpoint.
* */min_gap: the fp64 oracle's smallest relative top-k decision gap per config
  (tie rule); the oracle's beams are asserted identical to the
  reference's (tokens and fp64 log-probs bit for bit) before anything is saved.

Configs are drawn with the reference's own Rng (ksref_descriptors,
Rng::derive(2404, i)); tests check ks_synthetic_descriptors against them.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import OracleModel, RefModel  # noqa: E402
from paper_2404_10162_b200 import workloads as W  # noqa: E402

THREADS = os.cpu_count() or 1


def cfg2_indices():
    rng = np.random.default_rng(W.SEED)
    rest = np.sort(rng.choice(np.arange(4096, 65536), 4096, replace=False))
    return np.concatenate([np.arange(4096), rest]).astype(np.int64)


def decode_both(path, idx, k, greedy=False):
    o, r = OracleModel(path), RefModel(path)
    desc = r.descriptors(int(idx.max()) + 1, W.SEED)[idx]
    tok, bad = r.encode(desc)
    assert bad == 0, "descriptor outside the vocabulary"
    t0 = time.time()
    if greedy:
        ref = {"tokens": r.greedy(tok, THREADS)}
        ora = o.beam(tok, 1, None, [], threads=THREADS)
        assert (ora["tokens"][:, 0] == ref["tokens"]).all(), "oracle k=1 != reference greedy"
    else:
        ref = r.beam(tok, k, desc, W.reference_predicate_text(path), THREADS)
        h = W.read_header(path)
        preds = [o.membership(), o.budget({n: 1.0 for n in h["names"]}, W.BUDGETS[h["header"]["kernel"]])]
        ora = o.beam(tok, k, desc, preds, threads=THREADS)
        assert (ora["tokens"] == ref["tokens"]).all() and (ora["status"] == ref["status"]).all()
        assert np.array_equal(ora["log_prob"], ref["log_prob"]), "oracle lp != reference lp"
    print(f"  {len(idx)} configs, k={k}: {time.time() - t0:.0f} s, "
          f"tie-adjacent {(ora['min_gap'] < 1e-4).mean():.3f}", flush=True)
    out = {"index": idx, "desc": desc, "tok": tok, "min_gap": ora["min_gap"]}
    for key in ("tokens", "log_prob", "count", "status", "fail_step"):
        if key in ref:
            out[key] = ref[key]
    if not greedy:
        out["fail_pred"] = ora["fail_pred"]
    return out


def main():
    out = os.path.join(HERE, "baseline_parity.npz")
    only = sys.argv[1:]  # e.g. `cfg5`: regenerate that workload, keep the others
    fx = dict(np.load(out)) if only and os.path.exists(out) else {}
    want = lambda c: not only or c in only  # noqa: E731
    if want("cfg1"):
        print("cfg1", flush=True)
        for k, v in decode_both(W.DEFAULT_CKPT, np.arange(1000, dtype=np.int64), 1, greedy=True).items():
            fx[f"cfg1/{k}"] = v
    if want("cfg5"):
        print("cfg5", flush=True)
        p5 = W.cfg5_checkpoint_reference()
        fx["cfg5/sha256"] = np.array(W.sha256(p5))
        for k, v in decode_both(p5, np.arange(256, dtype=np.int64), 16).items():
            fx[f"cfg5/{k}"] = v
    if want("cfg2"):
        print("cfg2", flush=True)
        for k, v in decode_both(W.DEFAULT_CKPT, cfg2_indices(), 5).items():
            fx[f"cfg2/{k}"] = v
    np.savez_compressed(out, **fx)
    print("cfg5 sha256", fx["cfg5/sha256"], "(workloads.CFG5_SHA256)")


if __name__ == "__main__":
    main()
