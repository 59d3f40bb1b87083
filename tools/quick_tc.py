import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2404_10162_b200._cabi import Engine
from oracle.oracle import OracleModel
path = "tests/golden/_big/attn_default_trained.ckpt"
o = OracleModel(path)
rng = np.random.default_rng(0)
B = 65536
tok = np.stack([rng.integers(0, len(o.input_values[f]), B) for f in range(7)], 1).astype(np.int32)
preds = [o.membership(), o.budget({n: 1.0 for n in o.names}, 60.0)]
ref = None
for prec in sys.argv[1:]:
    e = Engine(path, 0, prec)
    e.beam(tok[:256], 5, None, preds)
    t0 = time.time(); g = e.beam(tok, 5, None, preds); t1 = time.time()
    print(f"{prec}: B={B} wall {t1-t0:.3f}s -> {B/(t1-t0):.0f} configs/s launches={e.launches()}", flush=True)
    e.profile_reset(True); e.beam(tok, 5, None, preds); ms, n, fl = e.profile(); e.profile_reset(False)
    print(f"  gemm {ms:.2f} ms over {n} launches, {fl/ms/1e9:.1f} TFLOP/s useful", flush=True)
    if ref is None:
        ref = g
    else:
        same = (g["tokens"] == ref["tokens"]).all(axis=(1, 2))
        top1 = (g["tokens"][:, 0] == ref["tokens"][:, 0]).all(axis=1)
        print(f"  vs {sys.argv[1]}: full-list agreement {same.mean()*100:.3f}%  top1 {top1.mean()*100:.3f}%  max|dlp| {np.nanmax(np.abs(np.where(np.isfinite(ref['log_prob']), g['log_prob']-ref['log_prob'], 0))):.2e}", flush=True)
