"""Shared test helpers (paths, parity rule)."""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIG_CKPT = os.path.join(ROOT, "tests", "golden", "attn_default_trained.ckpt")

# Tie rule: a config is tie-adjacent when two candidates whose
# order decides top-k membership or final rank are within this relative gap
# in the fp64 reference; decoded sequences must be identical on all others.
TIE_REL = 1e-4


def golden_path(name: str) -> str:
    return os.path.join(ROOT, "tests", "golden", name)


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def compare_beams(gpu, ora, lp_rel=1e-4, tie_rel=TIE_REL):
    """Returns (n_compared, n_tie_adjacent, mismatching rows) under the tie rule."""
    B = len(ora["count"])
    tie = ora["min_gap"] < tie_rel
    bad = []
    for b in range(B):
        if tie[b]:
            continue
        if gpu["status"][b] != ora["status"][b]:
            bad.append(b)
            continue
        if ora["status"][b] != 0:
            if gpu["fail_step"][b] != ora["fail_step"][b] or gpu["fail_pred"][b] != ora["fail_pred"][b]:
                bad.append(b)
            continue
        n = ora["count"][b]
        if gpu["count"][b] != n or not (gpu["tokens"][b, :n] == ora["tokens"][b, :n]).all():
            bad.append(b)
            continue
        lo, lg = ora["log_prob"][b, :n], gpu["log_prob"][b, :n]
        if not np.all(np.abs(lo - lg) <= lp_rel * np.maximum(np.abs(lo), 1.0)):
            bad.append(b)
    return B - int(tie.sum()), int(tie.sum()), bad
