import sys, numpy as np
sys.path.insert(0, '.')
from oracle.oracle import OracleModel
from tests.util import golden_path
from paper_2404_10162_b200._cabi import Engine
p = golden_path(sys.argv[1] + ".ckpt")
o = OracleModel(p)
e = Engine(p, 0, sys.argv[2] if len(sys.argv) > 2 else "f16x3")
rng = np.random.default_rng(1)
tok = np.stack([rng.integers(0, len(o.input_values[f]), 128) for f in range(7)], 1).astype(np.int32)
for k in (1, 2, 3, 8, 64):
    print("k", k, flush=True)
    g = e.beam(tok, k)
    a = o.beam(tok, k)
    print("match", (g["tokens"] == a["tokens"]).all(axis=(1, 2)).mean(), flush=True)
