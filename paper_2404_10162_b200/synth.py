"""Synthetic workloads for benchmarking: a randomly initialised model written
in the reference checkpoint format and problem descriptors drawn WITH
replacement from the synthetic grids (the reference grid has
only 46,656 unique points, so 64k / 1M workloads must resample).

The checkpoint follows init_model's shapes and initialiser families
(proj/src/models.cpp:178-259, proj/src/nn.cpp:299-321): LSTM weights
U(-1/sqrt(H), 1/sqrt(H)) with forget bias 1, dense weights Xavier-uniform,
zero dense biases.  Values come from numpy's PCG64, so the weights are not
bit-identical to the reference's init_model (throughput does not depend on
the weight values; parity runs use checkpoints written by the reference).
"""
from __future__ import annotations

import numpy as np

from .specs import BUILTIN_SPECS, FIELDS, input_grids


def _lstm(rng, prefix, n_in, H, t):
    lim = 1.0 / np.sqrt(H)
    for g in ("input", "forget", "output", "cand"):
        t[f"{prefix}.w_{g}"] = rng.uniform(-lim, lim, (n_in + H, H))
        t[f"{prefix}.b_{g}"] = np.full(H, 1.0 if g == "forget" else 0.0)


def _dense(rng, prefix, n_in, n_out, t):
    lim = np.sqrt(6.0 / (n_in + n_out))
    t[f"{prefix}.weights"] = rng.uniform(-lim, lim, (n_in, n_out))
    t[f"{prefix}.bias"] = np.zeros(n_out)


def write_checkpoint(path, kernel="ConvAsm1x1U", variant="attn", n_a=256, n_s=512, n_d=2,
                     e_size=256, seed=1, input_values=None, dropout=0.0, recurrent_dropout=0.0):
    spec = BUILTIN_SPECS[kernel]
    grids = input_values or input_grids(kernel)
    d_in = sum(len(g) for g in grids)
    d_fb = 1 + sum(len(v) for _, v in spec.params)
    rng = np.random.default_rng(seed)
    t = {}
    if variant in ("attn", "attn-2"):
        _lstm(rng, "pre.fwd", d_in, n_a, t)
        _lstm(rng, "pre.bwd", d_in, n_a, t)
        _lstm(rng, "post", 2 * n_a + (d_fb if variant == "attn" else 0), n_s, t)
        _dense(rng, "attn.hidden", n_s + 2 * n_a, n_d, t)
        _dense(rng, "attn.out", n_d, 1, t)
        head_in = n_s
    elif variant == "enc-dec":
        _lstm(rng, "encoder", d_in, e_size, t)
        _lstm(rng, "decoder", d_fb, e_size, t)
        head_in = e_size
    else:
        raise ValueError(f"variant {variant} not supported by the synthetic writer")
    for i, (_, vals) in enumerate(spec.params):
        _dense(rng, f"head.{i}", head_in, len(vals), t)
    lines = ["format: kernelseer-checkpoint/1", f"variant: {variant}", f"kernel: {kernel}",
             "precision: fp32", f"encoder_state_size: {e_size}", f"pre_attention_size: {n_a}",
             f"post_attention_size: {n_s}", f"attention_dense_nodes: {n_d}",
             "decoder_cell_size: 256", f"dropout: {dropout:g}", f"recurrent_dropout: {recurrent_dropout:g}",
             "conv_layers: 64,3,1;32,3,1"]
    for f, g in zip(FIELDS, grids):
        lines.append(f"input_vocab.{f}: " + ",".join(str(v) for v in g))
    lines.append(f"output_params: {len(spec.params)}")
    for i, (name, vals) in enumerate(spec.params):
        lines.append(f"param.{i}: {name} = " + ",".join(str(v) for v in vals))
    names = sorted(t)  # the reference writer emits std::map (alphabetical) order
    for n in names:
        a = np.atleast_2d(t[n]) if t[n].ndim == 2 else t[n]
        lines.append(f"tensor: {n} " + "x".join(str(d) for d in a.shape))
    with open(path, "wb") as fh:
        fh.write(("\n".join(lines) + "\n\n").encode())
        for n in names:
            fh.write(np.ascontiguousarray(t[n], "<f4").tobytes())
    return path


def descriptors(n, kernel="ConvAsm1x1U", seed=2404, input_values=None):
    """n descriptors (n x 7 int64), each field drawn uniformly with replacement."""
    grids = input_values or input_grids(kernel)
    rng = np.random.default_rng(seed)
    cols = [np.asarray(g, np.int64)[rng.integers(0, len(g), n)] for g in grids]
    return np.stack(cols, 1)
