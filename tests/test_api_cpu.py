"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/ks_b200.h declares; the reference-named
Python module exposes the binding surface; host logic that needs no GPU
(specs, checkpoints and their error kinds, predicate semantics, validate)."""
import json
import os
import re
import shutil
import tempfile

import pytest

from tests.util import ROOT, golden_path


def header_functions():
    text = open(os.path.join(ROOT, "include", "ks_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ks_[a-z0-9_]+)\s*\(", text)) - {"ks_host_pred_fn"})


def test_cabi_exports_every_declared_symbol():
    import ctypes

    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2404_10162_b200", "libks_b200.so"))
    names = header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_cabi_symbol_list_matches_python_binding():
    from paper_2404_10162_b200 import _cabi

    assert set(_cabi.EXPORTS) <= set(header_functions())


def test_builtin_specs_match_reference():
    import paper_2404_10162_b200 as ks

    ref = json.load(open(golden_path("builtin_specs.json")))
    got = ks.builtin_specs()
    assert [s.name for s in got] == [r["name"] for r in ref]
    for s, r in zip(got, ref):
        assert [[n, list(v)] for n, v in s.params] == r["params"]
        assert ks.search_space_size(s) == r["search_space"]
    # constraints_test.cpp:89-95 known answers
    assert ks.search_space_size(ks.builtin_spec("ConvAsm1x1U")) == 3440640
    assert ks.search_space_size(ks.builtin_spec("ConvAsmBwdWrW3x3")) == 20480
    with pytest.raises(ks.KernelseerError):
        ks.builtin_spec("Nope")


def test_load_checkpoint_metadata():
    import paper_2404_10162_b200 as ks

    p = ks.load_checkpoint(golden_path("attn_small_trained.ckpt"))
    assert p.kernel == "ConvAsm1x1U" and p.variant == "attn" and p.precision == "fp32"
    assert [n for n, _ in p.spec.params] == [n for n, _ in ks.builtin_spec("ConvAsm1x1U").params]


def _corrupt(src, dst, fn):
    raw = open(src, "rb").read()
    open(dst, "wb").write(fn(raw))
    return dst


@pytest.mark.parametrize("how,kind", [
    ("truncate", 1), ("extend", 2), ("version", 0), ("malformed", 3), ("missing", 4)])
def test_checkpoint_error_kinds(tmp_path, how, kind):
    """data_test.cpp:200-251: distinct CheckpointError kinds."""
    import ctypes

    import paper_2404_10162_b200 as ks
    from paper_2404_10162_b200 import _cabi

    src = golden_path("tiny_attn_s22.ckpt")
    dst = str(tmp_path / "bad.ckpt")
    if how == "truncate":
        _corrupt(src, dst, lambda r: r[:-4])
    elif how == "extend":
        _corrupt(src, dst, lambda r: r + b"\0\0\0\0")
    elif how == "version":
        _corrupt(src, dst, lambda r: r.replace(b"kernelseer-checkpoint/1", b"kernelseer-checkpoint/9", 1))
    elif how == "malformed":
        _corrupt(src, dst, lambda r: r.replace(b"variant: attn", b"variant attn", 1))
    else:
        dst = str(tmp_path / "absent.ckpt")
    with pytest.raises(ks.KernelseerError):
        ks.load_checkpoint(dst)
    L = _cabi.lib()
    h = ctypes.c_void_p()
    assert L.ks_checkpoint_load(dst.encode(), ctypes.byref(h)) == 6
    assert L.ks_checkpoint_error_kind() == kind


def test_predicate_factories_and_validate():
    import paper_2404_10162_b200 as ks

    spec = ks.builtin_spec("ConvAsmBwdWrW3x3")
    d = {"n": 32, "c": 64, "h": 14, "w": 14, "k": 64, "y": 3, "x": 3}
    full = {n: v[0] for n, v in spec.params}
    mem = ks.membership_predicate(spec)
    assert mem.name == "membership:ConvAsmBwdWrW3x3" and mem.device_evaluable
    assert ks.validate(spec, d, full, [mem]) is None
    bud = ks.resource_budget_predicate({"chunk_size": 1.0, "pipe_lines_depth": 2.0}, 9.0, "tight")
    assert ks.validate(spec, d, full, [mem, bud]) == {"predicate": "tight",
                                                     "params": ["chunk_size", "pipe_lines_depth"]}
    with pytest.raises(ks.KernelseerError):
        ks.resource_budget_predicate({"chunk_size": -1.0}, 5.0)
    with pytest.raises(ks.KernelseerError):
        ks.resource_budget_predicate({"chunk_size": 1.0}, -5.0)
    wg = ks.product_limit_predicate(["k_per_wave", "n_per_group"], 64, 1024, "workgroup")
    assert ks.validate(spec, d, dict(full, k_per_wave=8, n_per_group=2), [wg]) is None
    assert ks.validate(spec, d, dict(full, k_per_wave=8, n_per_group=4), [wg])["predicate"] == "workgroup"
    div = ks.divisibility_predicate([("k_per_wave", 4)], "tile")
    assert ks.validate(spec, d, dict(full, k_per_wave=8), [div]) is None
    assert ks.validate(spec, dict(d, k=12), dict(full, k_per_wave=8), [div])["predicate"] == "tile"
    opaque = ks.predicate("chunk16", lambda desc, p: p.get("chunk_size", 16) == 16)
    assert not opaque.device_evaluable
    assert ks.validate(spec, d, full, [opaque])["predicate"] == "chunk16"
