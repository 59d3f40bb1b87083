"""Drop-in boundary pieces that run without a GPU: workload descriptors drawn
with the reference's Rng, encode_problem's OOV / snap semantics
(proj/tests/encoding_test.cpp:132-146), the cfg5 checkpoint bytes, and the
reference arm's library isolation."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2404_10162_b200 import workloads as W
from tests.util import ROOT

ref = pytest.importorskip("oracle.oracle")
needs_ref = pytest.mark.skipif(not ref.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_synthetic_descriptors_are_the_reference_rng_draws():
    """ks_synthetic_descriptors (config i <- Rng::derive(2404, i)) equals the
    reference's own Rng over the model vocabulary, for the prefix and for
    slices anywhere in a 1M-config workload (per-config streams)."""
    from paper_2404_10162_b200 import _cabi

    r = ref.RefModel(W.DEFAULT_CKPT)
    iv = W.read_header(W.DEFAULT_CKPT)["inputs"]
    assert np.array_equal(_cabi.synthetic_descriptors(iv, 5000), r.descriptors(5000))
    for start in (4096, 65535, 1 << 19, (1 << 20) - 300):
        assert np.array_equal(_cabi.synthetic_descriptors(iv, 300, start=start),
                              r.descriptors(300, start=start))
    assert np.array_equal(_cabi.synthetic_descriptors(iv, 64, seed=7), r.descriptors(64, seed=7))


def test_synthetic_descriptors_match_the_committed_fixture():
    """Same draws as the configs the parity fixtures were decoded on."""
    import paper_2404_10162_b200 as ks

    fx = np.load(os.path.join(ROOT, "tests", "golden", "baseline_parity.npz"))
    params = ks.load_checkpoint(W.DEFAULT_CKPT)
    idx = fx["cfg2/index"]
    d = ks.synthetic_descriptors(params, int(idx.max()) + 1)
    assert np.array_equal(d[idx], fx["cfg2/desc"])
    assert np.array_equal(ks.synthetic_descriptors(params, 1000), fx["cfg1/desc"])


def test_encode_problem_oov_names_field_and_snaps():
    """encoding_test.cpp:132-146: an unseen value raises ValidationError naming
    the field and the nearest known value; allow_nearest snaps to it (ties to
    the smaller value, encoding.cpp:26-34)."""
    import paper_2404_10162_b200 as ks

    params = ks.load_checkpoint(W.DEFAULT_CKPT)
    d = {"n": 3, "c": 16, "h": 7, "w": 7, "k": 16, "y": 1, "x": 1}
    with pytest.raises(ks.KernelseerError) as e:
        ks.encode_problem(params, d)
    assert "field n" in str(e.value) and "nearest known: 2" in str(e.value)
    assert ks.encode_problem(params, d, snap=True) == [1, 0, 0, 0, 0, 0, 0]
    d2 = dict(d, n=1, w=1000)
    with pytest.raises(ks.KernelseerError, match="field w"):
        ks.encode_problem(params, d2)
    assert ks.encode_problem(params, d2, snap=True)[3] == 7


@needs_ref
def test_encode_problem_matches_reference_on_random_oov():
    import paper_2404_10162_b200 as ks

    params = ks.load_checkpoint(W.DEFAULT_CKPT)
    r = ref.RefModel(W.DEFAULT_CKPT)
    rng = np.random.default_rng(5)
    desc = np.stack([rng.integers(1, 1100, 400) for _ in range(5)] + [np.ones(400, np.int64)] * 2, 1)
    desc[::3, :5] = r.descriptors(400)[::3, :5]  # some rows in-vocabulary
    names = ["n", "c", "h", "w", "k", "y", "x"]
    for snap in (False, True):
        rt, rf = r.encode_ex(desc, snap)
        for b in range(len(desc)):
            dd = {n: int(v) for n, v in zip(names, desc[b])}
            if rf[b]:
                with pytest.raises(ks.KernelseerError, match=f"field {rf[b]} "):
                    ks.encode_problem(params, dd, snap=snap)
            else:
                assert ks.encode_problem(params, dd, snap=snap) == list(rt[b])


@needs_ref
def test_cfg5_checkpoint_bytes_equal_the_reference():
    """Our init_model + save_checkpoint (engine arm / GPU tests) and the
    reference's (fixtures, reference arm) write the same cfg5 file."""
    fx = np.load(os.path.join(ROOT, "tests", "golden", "baseline_parity.npz"))
    ours = W.cfg5_checkpoint_ours()
    assert W.sha256(ours) == str(fx["cfg5/sha256"]) == W.CFG5_SHA256


@needs_ref
def test_reference_arm_maps_no_engine_library():
    """bench.py --impl reference runs the unmodified reference only."""
    code = ("import bench, sys; sys.argv=['bench.py']; bench.W = bench.WORKLOADS['cfg1'];"
            "import paper_2404_10162_b200.workloads, paper_2404_10162_b200.specs;"
            "from oracle.oracle import RefModel; RefModel(paper_2404_10162_b200.workloads.DEFAULT_CKPT);"
            "bench.assert_no_engine_mapped(); print('clean')")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "clean" in out.stdout, out.stderr
