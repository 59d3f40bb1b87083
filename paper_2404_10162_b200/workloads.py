"""The BASELINE.json workloads, defined once for bench.py (both arms) and the
parity tests.  Pure Python: importing this module maps no engine library (the
reference arm of bench.py relies on that).

* Models.  cfg1-cfg3: the tracked default-size ``attn`` checkpoint
  ``tests/golden/attn_default_trained.ckpt`` (n_a=256, n_s=512, n_d=2,
  ConvAsm1x1U), trained by the reference itself with the recipe of SURVEY.md
  §8(a) (``tests/golden/make_fixtures.py --big``).  cfg5: n_a = n_s = 1024,
  ConvAsmBwdWrW1x1, the reference's ``init_model(seed 1)`` with every head
  weight scaled by 2^8 (exact in fp32) so decisions are not tie-dominated;
  written by our byte-identical ``init_model`` (engine arm) or the reference's
  own (reference arm, parity fixtures) -- ``CFG5_SHA256`` pins the bytes.
* Configs.  Config i of a workload is ``Rng::derive(2404, i)``'s draw over the
  model's input vocabulary (``ks_synthetic_descriptors``; the reference arm and
  the fixtures draw with the reference's own Rng), so the first 4,096 configs
  of cfg2 are exactly the parity-fixture prefix.
* Predicates.  ``membership_predicate(spec)`` + ``resource_budget_predicate(
  {every param: 1.0}, budget)``.
"""
from __future__ import annotations

import hashlib
import os
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEFAULT_CKPT = os.path.join(ROOT, "tests", "golden", "attn_default_trained.ckpt")
SEED = 2404
HEAD_SCALE = 256.0  # 2^8: exact fp32 scaling of the cfg5 head weights
CFG5 = dict(kernel="ConvAsmBwdWrW1x1", n_a=1024, n_s=1024, n_d=2, init_seed=1)
# sha256 of the cfg5 checkpoint as the reference writes it (ref init_model +
# save_checkpoint, heads x HEAD_SCALE); tests/golden/make_baseline_fixtures.py
CFG5_SHA256 = "0d57b9379219260d5dcfd74a27fcfdec8d93a670d6a4b231ce9ee28359432745"

# budget of the resource_budget predicate per workload kernel: sum of values <= B
BUDGETS = {"ConvAsm1x1U": 60.0, "ConvAsmBwdWrW1x1": 40.0}

WORKLOADS = {
    "cfg1": dict(model="default", beam=1, configs=1000, greedy=True,
                 label="BASELINE config 1: greedy decode of 1k configs"),
    "cfg2": dict(model="default", beam=5, configs=65536, greedy=False,
                 label="BASELINE config 2: constrained beam search beam=5, 64k configs on 1 B200"),
    "cfg3": dict(model="default", beam=5, configs=1 << 20, greedy=False,
                 label="BASELINE config 3: constrained beam search beam=5, 1M configs sharded across GPUs"),
    "cfg5": dict(model="cfg5", beam=16, configs=16384, greedy=False,
                 label="BASELINE config 5 shape: n_a=n_s=1024 (1 layer; the reference has no layer count), "
                       "beam=16, ConvAsmBwdWrW1x1"),
}


def read_header(path):
    with open(path, "rb") as f:
        head = f.read(1 << 16).split(b"\n\n")[0].decode().split("\n")
    kv = {}
    names, values, inputs = [], [], []
    for line in head:
        k, _, v = line.partition(": ")
        if k.startswith("param."):
            n, _, vals = v.partition(" = ")
            names.append(n)
            values.append([int(x) for x in vals.split(",")])
        elif k.startswith("input_vocab."):
            inputs.append([int(x) for x in v.split(",")])
        elif k != "tensor":
            kv[k] = v
    return {"header": kv, "names": names, "values": values, "inputs": inputs}


def scale_heads(src, dst, scale=HEAD_SCALE):
    """Copies a checkpoint with every head.<p>.weights tensor multiplied by
    `scale` (a power of two: exact in fp32)."""
    raw = open(src, "rb").read()
    sep = raw.index(b"\n\n")
    header = raw[:sep].decode().split("\n")
    payload = bytearray(raw[sep + 2:])
    off = 0
    for line in header:
        if not line.startswith("tensor: "):
            continue
        name, shape = line[8:].rsplit(" ", 1)
        n = int(np.prod([int(d) for d in shape.split("x")]))
        if name.startswith("head.") and name.endswith(".weights"):
            a = np.frombuffer(bytes(payload[off:off + 4 * n]), "<f4") * np.float32(scale)
            payload[off:off + 4 * n] = a.astype("<f4").tobytes()
        off += 4 * n
    with open(dst, "wb") as f:
        f.write(raw[:sep + 2])
        f.write(bytes(payload))
    return dst


def sha256(path):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for blk in iter(lambda: f.read(1 << 20), b""):
            h.update(blk)
    return h.hexdigest()


def grid_samples(ks, spec, kernel):
    """Samples whose descriptors cover every value of the synthetic grids, so
    build_vocab yields the full input vocabulary generate_synthetic's 5,000
    samples do (data.cpp:355-358; checked by the checkpoint hash)."""
    from .specs import input_grids

    grids = input_grids(kernel)
    fields = ["n", "c", "h", "w", "k", "y", "x"]
    params = {name: vals[0] for name, vals in ((p.name, p.values) for p in spec.params)} \
        if hasattr(spec.params[0], "name") else {n: v[0] for n, v in spec.params}
    out = []
    for j in range(max(len(g) for g in grids)):
        d = {f: g[j % len(g)] for f, g in zip(fields, grids)}
        out.append(ks.Sample(d, params, kernel))
    return out


def cfg5_checkpoint_ours(path=None):
    """cfg5 model written by OUR init_model / save_checkpoint (byte-identical to
    the reference's, tests/test_trainloop.py) with the heads scaled."""
    import paper_2404_10162_b200 as ks

    path = path or os.path.join(tempfile.gettempdir(), "ks_cfg5_attn1024_wrw1x1.ckpt")
    if os.path.exists(path) and (CFG5_SHA256 is None or sha256(path) == CFG5_SHA256):
        return path
    spec = ks.builtin_spec(CFG5["kernel"])
    cfg = ks.ModelConfig(variant="attn", pre_attention_size=CFG5["n_a"], post_attention_size=CFG5["n_s"],
                         attention_dense_nodes=CFG5["n_d"], dropout=0.0, recurrent_dropout=0.0)
    tmp = path + f".{os.getpid()}.raw"
    ks.save_checkpoint(ks.init_model(cfg, spec, grid_samples(ks, spec, CFG5["kernel"]), seed=CFG5["init_seed"]), tmp)
    scale_heads(tmp, path + f".{os.getpid()}")
    os.remove(tmp)
    os.replace(path + f".{os.getpid()}", path)
    if CFG5_SHA256 is not None and sha256(path) != CFG5_SHA256:
        raise RuntimeError("cfg5 checkpoint differs from the reference-written one")
    return path


def cfg5_checkpoint_reference(path=None):
    """cfg5 model written by the REFERENCE's init_model / save_checkpoint
    (oracle/_ref; test infrastructure and the reference arm only)."""
    from oracle.oracle import ref_init_save

    path = path or os.path.join(tempfile.gettempdir(), "ks_cfg5_attn1024_wrw1x1.ref.ckpt")
    if os.path.exists(path):
        return path
    tmp = path + f".{os.getpid()}.raw"
    ref_init_save(tmp, variant="attn", e_size=256, n_a=CFG5["n_a"], n_s=CFG5["n_s"], n_d=CFG5["n_d"], cell=256,
                  kernel=CFG5["kernel"], synth_count=5000, synth_seed=7, init_seed=CFG5["init_seed"])
    scale_heads(tmp, path + f".{os.getpid()}")
    os.remove(tmp)
    os.replace(path + f".{os.getpid()}", path)
    return path


def train_checkpoint(reference=False, path=None):
    """BASELINE config 4's model: the default attn model (n_a=256, n_s=512, n_d=2,
    ConvAsm1x1U) from init_model(seed 1) with the ModelConfig default dropout
    0.2 / recurrent 0.2 (models.hpp:28-41), written by our init_model or the
    reference's (identical bytes)."""
    path = path or os.path.join(tempfile.gettempdir(),
                                "ks_train_attn256_512_d0.2" + (".ref" if reference else "") + ".ckpt")
    if os.path.exists(path):
        return path
    tmp = path + f".{os.getpid()}.raw"
    if reference:
        from oracle.oracle import ref_init_save

        ref_init_save(tmp, variant="attn", e_size=256, n_a=256, n_s=512, n_d=2, cell=256, kernel="ConvAsm1x1U",
                      synth_count=5000, synth_seed=7, init_seed=1)
    else:
        import paper_2404_10162_b200 as ks

        spec = ks.builtin_spec("ConvAsm1x1U")
        cfg = ks.ModelConfig(variant="attn", dropout=0.0, recurrent_dropout=0.0)
        ks.save_checkpoint(ks.init_model(cfg, spec, grid_samples(ks, spec, "ConvAsm1x1U"), seed=1), tmp)
    raw = open(tmp, "rb").read()
    os.remove(tmp)
    raw = raw.replace(b"\ndropout: 0\nrecurrent_dropout: 0\n", b"\ndropout: 0.2\nrecurrent_dropout: 0.2\n", 1)
    with open(path + f".{os.getpid()}", "wb") as f:
        f.write(raw)
    os.replace(path + f".{os.getpid()}", path)
    return path


def predicate_dicts(path):
    """membership + budget as C-ABI predicate dicts (paper_2404_10162_b200._cabi.pack_preds)."""
    h = read_header(path)
    kernel = h["header"]["kernel"]
    names, values = h["names"], h["values"]
    srt = sorted(names)
    return [{"kind": 1, "allowed": np.ones(sum(len(v) for v in values), np.uint8)},
            {"kind": 2, "term_pos": np.array([names.index(n) for n in srt], np.int32),
             "term_w": np.ones(len(srt)), "budget": BUDGETS[kernel]}]


def reference_predicate_text(path):
    """The same predicates in ref_shim's text form (oracle.oracle.RefModel.beam)."""
    h = read_header(path)
    budget = BUDGETS[h["header"]["kernel"]]
    return "membership\nbudget bud %g " % budget + ",".join(f"{n}=1.0" for n in h["names"])
