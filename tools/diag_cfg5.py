"""Diagnostic: cfg5 mismatches vs the reference fixture (gaps, lp deltas)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2404_10162_b200 import workloads as W
from paper_2404_10162_b200._cabi import Engine
from tests.util import compare_beams

fx = dict(np.load("tests/golden/baseline_parity.npz"))
r = {k.split("/", 1)[1]: v for k, v in fx.items() if k.startswith("cfg5/")}
path = W.cfg5_checkpoint_ours()
for prec in sys.argv[1:] or ["f16x3", "fp32"]:
    g = Engine(path, 0, prec).beam(r["tok"], 16, r["desc"], W.predicate_dicts(path))
    n, ties, bad = compare_beams(g, r)
    print(prec, "compared", n, "ties", ties, "bad", bad)
    for b in bad:
        same = (g["tokens"][b] == r["tokens"][b]).all(axis=1)
        first = int(np.argmin(same)) if not same.all() else -1
        print(f"  cfg {b}: min_gap {r['min_gap'][b]:.3e} first differing rank {first} "
              f"count {g['count'][b]}/{r['count'][b]}")
        print("    ref lp", np.round(r["log_prob"][b][:16], 6))
        print("    gpu lp", np.round(g["log_prob"][b][:16], 6))
        d = np.abs(g["log_prob"][b] - r["log_prob"][b])
        print("    max |dlp| on equal ranks", d[same].max() if same.any() else None)
