"""Generates tests/golden/train_golden.npz with the UNMODIFIED reference
(oracle/_ref/libkernelseer_ref.so, built by `make -C oracle ref` from
/root/reference/proj/src; driven through oracle/ref_shim.cpp):

* Rng streams: Rng::derive(seed, stream).uniform() and train_model's
  per-epoch shuffle (proj/include/kernelseer/rng.hpp, proj/src/models.cpp:895-900);
* for the tiny enc-dec / attn / attn-2 fixtures (committed *.ckpt), with and
  without dropout: the summed teacher-forced loss and flat gradients of a
  16-sample batch (model_loss_gradients, models.cpp:788-797, per-sample dropout
  streams as train_model draws them), and the parameters after each of 3
  optimiser steps (train_model's batch body: / batch, clip_global_norm 5.0,
  adam_step lr 3e-3; models.cpp:905-947).

    make -C oracle ref && python tests/golden/make_train_fixtures.py
"""
import ctypes as C
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

TRAIN_MODELS = ["tiny_attn_s3423", "tiny_attn2_s3423", "tiny_encdec_s3423", "tiny_attn_s232"]
DROPOUT = (0.3, 0.2)
RNG_CASES = [(1, 0, 20), (7, 5, 700), (2404, (3 << 32) | 17, 40)]
SHUFFLE_CASES = [(1, 1, 10), (1, 4, 33), (99, 2, 1000)]
B = 16
STEPS = 3
LR = 3e-3


def with_dropout(src, dst, rates=DROPOUT):
    """The same checkpoint with `dropout` / `recurrent_dropout` set in its header."""
    raw = open(src, "rb").read()
    sep = raw.index(b"\n\n")
    lines = raw[:sep].decode().split("\n")
    lines = [f"dropout: {rates[0]}" if l.startswith("dropout:") else
             f"recurrent_dropout: {rates[1]}" if l.startswith("recurrent_dropout:") else l for l in lines]
    with open(dst, "wb") as f:
        f.write(("\n".join(lines)).encode() + raw[sep:])
    return dst


def batch(ck, seed):
    rng = np.random.default_rng(seed)
    tok = np.stack([rng.integers(0, len(ck.inputs[f]), B) for f in range(7)], 1).astype(np.int32)
    tgt = np.stack([rng.integers(0, v, B) for v in ck.vsizes], 1).astype(np.int32)
    idx = rng.permutation(1000)[:B].astype(np.int64)
    return tok, tgt, idx


def ref_lib():
    from oracle.oracle import rlib

    L = rlib()
    P = C.POINTER
    L.ksref_num_params.restype = C.c_int64
    L.ksref_num_params.argtypes = [C.c_void_p]
    L.ksref_get_params.argtypes = [C.c_void_p, P(C.c_double)]
    L.ksref_loss_grads.argtypes = [C.c_void_p, P(C.c_int32), P(C.c_int32), C.c_int64, C.c_int, C.c_int64,
                                   C.c_uint64, P(C.c_int64), P(C.c_double), P(C.c_double)]
    L.ksref_trainer_new.restype = C.c_void_p
    L.ksref_trainer_new.argtypes = [C.c_double]
    L.ksref_trainer_free.argtypes = [C.c_void_p]
    L.ksref_train_step.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int32), P(C.c_int32), C.c_int64, C.c_int,
                                   C.c_int64, C.c_uint64, P(C.c_int64), C.c_double, P(C.c_double)]
    L.ksref_uniforms.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, P(C.c_double)]
    L.ksref_shuffle.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, P(C.c_int64)]
    L.ksref_load.restype = C.c_void_p
    L.ksref_load.argtypes = [C.c_char_p]
    L.ksref_free.argtypes = [C.c_void_p]
    return L


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


def ref_loss_grads(L, path, tok, tgt, epoch=-1, seed=0, idx=None, threads=4):
    h = L.ksref_load(path.encode())
    g = np.zeros(L.ksref_num_params(h))
    loss = C.c_double()
    rc = L.ksref_loss_grads(h, _p(tok, C.c_int32), _p(tgt, C.c_int32), len(tok), threads, epoch, seed,
                            _p(idx, C.c_int64), C.byref(loss), _p(g, C.c_double))
    L.ksref_free(h)
    assert rc == 0
    return loss.value, g


def ref_train(L, path, tok, tgt, steps, epoch0, seed, idx, lr=LR, clip=5.0, threads=4):
    h = L.ksref_load(path.encode())
    tr = L.ksref_trainer_new(lr)
    out, losses = [], []
    for s in range(steps):
        loss = C.c_double()
        rc = L.ksref_train_step(h, tr, _p(tok, C.c_int32), _p(tgt, C.c_int32), len(tok), threads, epoch0 + s,
                                seed, _p(idx, C.c_int64), clip, C.byref(loss))
        assert rc == 0
        p = np.zeros(L.ksref_num_params(h))
        L.ksref_get_params(h, _p(p, C.c_double))
        out.append(p)
        losses.append(loss.value)
    L.ksref_trainer_free(tr)
    L.ksref_free(h)
    return np.stack(out), np.array(losses)


def main():
    from oracle.train_oracle import Checkpoint

    L = ref_lib()
    g = {}
    for seed, stream, n in RNG_CASES:
        u = np.zeros(n)
        L.ksref_uniforms(seed, stream, n, _p(u, C.c_double))
        g[f"rng/{seed}/{stream}"] = u
    for seed, epoch, n in SHUFFLE_CASES:
        o = np.zeros(n, np.int64)
        L.ksref_shuffle(seed, epoch, n, _p(o, C.c_int64))
        g[f"shuffle/{seed}/{epoch}/{n}"] = o
    with tempfile.TemporaryDirectory() as tmp:
        for stem in TRAIN_MODELS:
            for drop in (False, True):
                path = os.path.join(HERE, stem + ".ckpt")
                if drop:
                    path = with_dropout(path, os.path.join(tmp, stem + "_drop.ckpt"))
                ck = Checkpoint(path)
                tok, tgt, idx = batch(ck, 5)
                key = f"{stem}/{'drop' if drop else 'nodrop'}"
                loss, grads = ref_loss_grads(L, path, tok, tgt, epoch=2 if drop else -1, seed=11, idx=idx)
                g[key + "/tok"], g[key + "/tgt"], g[key + "/idx"] = tok, tgt, idx
                g[key + "/loss"], g[key + "/grads"] = np.array(loss), grads
                params, losses = ref_train(L, path, tok, tgt, STEPS, 1, 11, idx)
                g[key + "/train_params"], g[key + "/train_loss"] = params, losses
    np.savez_compressed(os.path.join(HERE, "train_golden.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
