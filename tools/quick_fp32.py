import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2404_10162_b200._cabi import Engine
from oracle.oracle import OracleModel
path = "tests/golden/_big/attn_default_trained.ckpt"
o = OracleModel(path)
e = Engine(path, 0, "fp32")
rng = np.random.default_rng(0)
for B in (4096, 65536):
    tok = np.stack([rng.integers(0, len(o.input_values[f]), B) for f in range(7)], 1).astype(np.int32)
    preds = [o.membership(), o.budget({n: 1.0 for n in o.names}, 60.0)]
    e.beam(tok[:256], 5, None, preds)
    t0 = time.time(); g = e.beam(tok, 5, None, preds); t1 = time.time()
    print(f"B={B} fp32 wall {t1-t0:.3f}s -> {B/(t1-t0):.0f} configs/s launches={e.launches()}", flush=True)
    e.profile_reset(True); e.beam(tok, 5, None, preds); ms, n, fl = e.profile(); e.profile_reset(False)
    print(f"  gemm {ms:.2f} ms over {n} launches, {fl/ms/1e9:.1f} TFLOP/s useful", flush=True)
