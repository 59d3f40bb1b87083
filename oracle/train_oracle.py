"""TEST INFRASTRUCTURE ONLY -- fp64 numpy restatement of the reference's
teacher-forced training step, the checker for the CUDA trainer.

Restates, batched over samples (one row per sample, same arithmetic per row):

* ``build_loss_graph`` for the enc-dec / attn / attn-2 variants
  (proj/src/models.cpp:638-780): bi-LSTM encoder over the 7 one-hot input
  steps, additive attention (models.cpp:700-712, the tape form of
  attention_weights / context_vector, models.cpp:265-294), the post-attention
  LSTM with teacher feedback one-hots, per-position heads and
  ``cross_entropy_logits``, loss = mean over positions (``sum_scaled``).
* ``Tape::backward`` for those ops (proj/src/autodiff.cpp:326-544): the LSTM
  cell (tape_lstm_step, models.cpp:578-593), softmax, weighted_sum, dense.
* variational dropout exactly as train_model draws it: per sample
  Rng::derive(seed, epoch << 32 | idx) (models.cpp:915-918) ->
  LstmMasks::make (models.cpp:559-573), through the C restatement of the Rng
  (ks_oracle.c, kso_dropout_masks).
* the optimiser step of train_model (models.cpp:943-947): grads / batch,
  ``clip_global_norm`` (nn.cpp:286-297), ``adam_step`` (nn.cpp:262-284).

Pinned against the unmodified reference (oracle/ref_shim.cpp
ksref_loss_grads / ksref_train_step) by tests/test_train_oracle_pin.py and the
committed fixtures tests/golden/train_golden.npz.  Only tests/ and bench.py's
reference leg may import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np

FIELDS = ["n", "c", "h", "w", "k", "y", "x"]
GATES = ["input", "forget", "output", "cand"]


def sig(x):
    return 1.0 / (1.0 + np.exp(-x))


class Checkpoint:
    """kernelseer-checkpoint/1 reader (proj/src/data.cpp:513-665, docs/formats.md:53-93)."""

    def __init__(self, path: str):
        raw = open(path, "rb").read()
        end = raw.index(b"\n\n")
        header = raw[:end].decode().split("\n")
        self.header, self.shapes, self.order = {}, {}, []
        self.outputs = []
        for line in header:
            key, _, val = line.partition(": ")
            if key == "tensor":
                name, dims = val.rsplit(" ", 1)
                self.shapes[name] = tuple(int(d) for d in dims.split("x"))
                self.order.append(name)
            elif key.startswith("param."):
                name, _, vals = val.partition(" = ")
                self.outputs.append((name, [int(v) for v in vals.split(",")]))
            else:
                self.header[key] = val
        off = end + 2
        self.tensors = {}
        for name in self.order:
            n = int(np.prod(self.shapes[name]))
            a = np.frombuffer(raw, "<f4", n, off).astype(np.float64)
            self.tensors[name] = a.reshape(self.shapes[name])
            off += 4 * n
        self.variant = self.header["variant"]
        self.inputs = [[int(v) for v in self.header["input_vocab." + f].split(",")] for f in FIELDS]
        self.n_a = int(self.header["pre_attention_size"])
        self.n_s = int(self.header["post_attention_size"])
        self.n_d = int(self.header["attention_dense_nodes"])
        self.e = int(self.header["encoder_state_size"])
        self.dropout = float(self.header.get("dropout", "0"))
        self.rdropout = float(self.header.get("recurrent_dropout", "0"))
        self.T = len(self.outputs)
        self.vsizes = [len(v) for _, v in self.outputs]
        self.in_off = np.cumsum([0] + [len(v) for v in self.inputs])[:-1]
        self.d_in = sum(len(v) for v in self.inputs)
        self.fb_off = np.cumsum([1] + self.vsizes)[:-1]
        self.d_fb = 1 + sum(self.vsizes)

    def flat(self, tensors=None) -> np.ndarray:
        t = self.tensors if tensors is None else tensors
        return np.concatenate([t[n].reshape(-1) for n in self.order])

    def unflat(self, v: np.ndarray) -> dict:
        out, o = {}, 0
        for n in self.order:
            k = int(np.prod(self.shapes[n]))
            out[n] = v[o:o + k].reshape(self.shapes[n]).copy()
            o += k
        return out


def _okso():
    from oracle.oracle import lib

    L = lib()
    L.kso_dropout_masks.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_double,
                                    C.POINTER(C.c_double)]
    L.kso_shuffle.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(C.c_int64)]
    L.kso_uniforms.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(C.c_double)]
    return L


def dropout_masks(ck: Checkpoint, seed: int, epoch: int, idx) -> tuple[np.ndarray, np.ndarray] | None:
    """Per-sample (input, recurrent) masks of the decoder LSTM, or None when
    dropout is off (LstmMasks::make returns inactive masks)."""
    if ck.dropout == 0.0 and ck.rdropout == 0.0:
        return None
    if ck.variant == "enc-dec":
        n_in, n_rec = ck.d_fb, ck.e
    else:
        n_in = 2 * ck.n_a + (ck.d_fb if ck.variant == "attn" else 0)
        n_rec = ck.n_s
    L = _okso()
    mi = np.zeros((len(idx), n_in))
    mr = np.zeros((len(idx), n_rec))
    buf = np.zeros(n_in + n_rec)
    for b, i in enumerate(idx):
        L.kso_dropout_masks(seed, (epoch << 32) | int(i), n_in, ck.dropout, n_rec, ck.rdropout,
                            buf.ctypes.data_as(C.POINTER(C.c_double)))
        mi[b], mr[b] = buf[:n_in], buf[n_in:]
    return mi, mr


def shuffle(seed: int, epoch: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.int64)
    _okso().kso_shuffle(seed, epoch, n, out.ctypes.data_as(C.POINTER(C.c_int64)))
    return out


# ---------------------------------------------------------------------------
# building blocks: forward returns a cache, backward accumulates into grads
# ---------------------------------------------------------------------------
class _Lstm:
    def __init__(self, P, G, prefix):
        self.W = [P[f"{prefix}.w_{g}"] for g in GATES]
        self.b = [P[f"{prefix}.b_{g}"] for g in GATES]
        self.gW = [G[f"{prefix}.w_{g}"] for g in GATES]
        self.gb = [G[f"{prefix}.b_{g}"] for g in GATES]
        self.H = self.b[0].shape[0]

    def fwd(self, x, h, c):
        xh = np.concatenate([x, h], 1)
        zi, zf, zo, zg = (xh @ W + b for W, b in zip(self.W, self.b))
        i, f, o, g = sig(zi), sig(zf), sig(zo), np.tanh(zg)
        c2 = f * c + i * g
        h2 = o * np.tanh(c2)
        return h2, c2, (xh, i, f, o, g, c, c2)

    def bwd(self, cache, dh, dc_next):
        xh, i, f, o, g, c, c2 = cache
        tc = np.tanh(c2)
        do = dh * tc
        dc = dc_next + dh * o * (1.0 - tc * tc)
        dz = [dc * g * i * (1.0 - i), dc * c * f * (1.0 - f), do * o * (1.0 - o), dc * i * (1.0 - g * g)]
        dxh = 0.0
        for k in range(4):
            self.gW[k] += xh.T @ dz[k]
            self.gb[k] += dz[k].sum(0)
            dxh = dxh + dz[k] @ self.W[k].T
        Kx = xh.shape[1] - self.H
        return dxh[:, :Kx], dxh[:, Kx:], dc * f


def _onehot(slots, width):
    out = np.zeros((len(slots), width))
    out[np.arange(len(slots)), slots] = 1.0
    return out


def loss_and_grads(ck: Checkpoint, P: dict, tok: np.ndarray, tgt: np.ndarray, masks=None,
                   want_logits=False):
    """Sum over the batch of the per-sample teacher-forced loss and of its
    parameter gradients (model_loss_gradients summed over samples).
    Returns (loss_sum, grads dict, per-position argmax matches)."""
    tok = np.asarray(tok, np.int64).reshape(-1, 7)
    tgt = np.asarray(tgt, np.int64).reshape(len(tok), ck.T)
    B, T = len(tok), ck.T
    G = {n: np.zeros_like(v) for n, v in P.items()}
    xs = [_onehot(ck.in_off[f] + tok[:, f], ck.d_in) for f in range(7)]
    fb = [_onehot(np.full(B, 0) if p == 0 else ck.fb_off[p - 1] + tgt[:, p - 1], ck.d_fb) for p in range(T)]
    mi, mr = masks if masks is not None else (None, None)
    feats, caches = [], []
    v = ck.variant
    if v == "enc-dec":
        enc = _Lstm(P, G, "encoder")
        dec = _Lstm(P, G, "decoder")
        h = np.zeros((B, ck.e))
        c = np.zeros((B, ck.e))
        ecache = []
        for f in range(7):
            h, c, cc = enc.fwd(xs[f], h, c)
            ecache.append(cc)
        for p in range(T):
            x = fb[p] if mi is None else fb[p] * mi
            hin = h if mr is None else h * mr
            h, c, cc = dec.fwd(x, hin, c)
            caches.append(cc)
            feats.append(h)
    elif v in ("attn", "attn-2"):
        pf, pb = _Lstm(P, G, "pre.fwd"), _Lstm(P, G, "pre.bwd")
        na, ns, nd = ck.n_a, ck.n_s, ck.n_d
        hf = [None] * 7
        hb = [None] * 7
        cf, cb = [None] * 7, [None] * 7
        h = np.zeros((B, na))
        c = np.zeros((B, na))
        for t in range(7):
            h, c, cf[t] = pf.fwd(xs[t], h, c)
            hf[t] = h
        h = np.zeros((B, na))
        c = np.zeros((B, na))
        for t in range(6, -1, -1):
            h, c, cb[t] = pb.fwd(xs[t], h, c)
            hb[t] = h
        A = np.stack([np.concatenate([hf[t], hb[t]], 1) for t in range(7)], 1)  # B x 7 x 2na
        Wh, bh = P["attn.hidden.weights"], P["attn.hidden.bias"]
        wo, bo = P["attn.out.weights"][:, 0], P["attn.out.bias"][0]
        Ws, Wa = Wh[:ns], Wh[ns:]
        post = _Lstm(P, G, "post")
        h = np.zeros((B, ns))
        c = np.zeros((B, ns))
        acache = []
        for p in range(T):
            pre = (h @ Ws)[:, None, :] + A @ Wa + bh  # B x 7 x nd
            hid = np.tanh(pre)
            e = hid @ wo + bo
            e = e - e.max(1, keepdims=True)
            al = np.exp(e)
            al = al / al.sum(1, keepdims=True)
            ctx = (al[:, :, None] * A).sum(1)
            x = np.concatenate([ctx, fb[p]], 1) if v == "attn" else ctx
            if mi is not None:
                x = x * mi
            hin = h if mr is None else h * mr
            acache.append((h, hid, al))
            h, c, cc = post.fwd(x, hin, c)
            caches.append(cc)
            feats.append(h)
    else:
        raise NotImplementedError(f"training oracle: variant {v}")

    # heads + cross entropy (sum_scaled 1/T)
    loss = 0.0
    matches = 0
    dfeat = []
    for p in range(T):
        W, b = P[f"head.{p}.weights"], P[f"head.{p}.bias"]
        lg = feats[p] @ W + b
        m = lg.max(1, keepdims=True)
        ex = np.exp(lg - m)
        s = ex.sum(1, keepdims=True)
        loss += float((-(lg[np.arange(B), tgt[:, p]] - m[:, 0] - np.log(s[:, 0]))).sum()) / T
        matches += int((lg.argmax(1) == tgt[:, p]).sum())
        d = ex / s
        d[np.arange(B), tgt[:, p]] -= 1.0
        d /= T
        G[f"head.{p}.weights"] += feats[p].T @ d
        G[f"head.{p}.bias"] += d.sum(0)
        dfeat.append(d @ W.T)

    if v == "enc-dec":
        dh = np.zeros((B, ck.e))
        dc = np.zeros((B, ck.e))
        for p in range(T - 1, -1, -1):
            _, dhin, dc = dec.bwd(caches[p], dh + dfeat[p], dc)
            dh = dhin if mr is None else dhin * mr
        for f in range(6, -1, -1):
            _, dh, dc = enc.bwd(ecache[f], dh, dc)
    else:
        dA = np.zeros_like(A)
        dh = np.zeros((B, ns))
        dc = np.zeros((B, ns))
        gWh = G["attn.hidden.weights"]
        for p in range(T - 1, -1, -1):
            dx, dhin, dc = post.bwd(caches[p], dh + dfeat[p], dc)
            if mi is not None:
                dx = dx * mi
            dh = dhin if mr is None else dhin * mr
            dctx = dx[:, :2 * na]
            s, hid, al = acache[p]
            dal = (dctx[:, None, :] * A).sum(2)
            dA += al[:, :, None] * dctx[:, None, :]
            de = al * (dal - (al * dal).sum(1, keepdims=True))
            G["attn.out.weights"][:, 0] += (hid * de[:, :, None]).sum((0, 1))
            G["attn.out.bias"][0] += de.sum()
            dpre = de[:, :, None] * wo[None, None, :] * (1.0 - hid * hid)
            gWh[:ns] += s.T @ dpre.sum(1)
            gWh[ns:] += np.einsum("bta,btd->ad", A, dpre)
            G["attn.hidden.bias"] += dpre.sum((0, 1))
            dh = dh + dpre.sum(1) @ Ws.T
            dA += dpre @ Wa.T
        dh = np.zeros((B, na))
        dc = np.zeros((B, na))
        for t in range(6, -1, -1):
            _, dh, dc = pf.bwd(cf[t], dh + dA[:, t, :na], dc)
        dh = np.zeros((B, na))
        dc = np.zeros((B, na))
        for t in range(7):
            _, dh, dc = pb.bwd(cb[t], dh + dA[:, t, na:], dc)
    return loss, G, matches


class Adam:
    """nn::adam_step + AdamConfig defaults (nn.hpp:96-101, nn.cpp:262-284)."""

    def __init__(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lr, self.b1, self.b2, self.eps = lr, beta1, beta2, eps
        self.m = self.v = None
        self.step = 0

    def apply(self, p: np.ndarray, g: np.ndarray):
        if self.m is None:
            self.m, self.v = np.zeros_like(p), np.zeros_like(p)
        self.step += 1
        bc1 = 1.0 - self.b1 ** self.step
        bc2 = 1.0 - self.b2 ** self.step
        self.m = self.b1 * self.m + (1.0 - self.b1) * g
        self.v = self.b2 * self.v + (1.0 - self.b2) * g * g
        return p - self.lr * (self.m / bc1) / (np.sqrt(self.v / bc2) + self.eps)


def clip_global_norm(g: np.ndarray, max_norm: float) -> np.ndarray:
    n = float(np.sqrt((g * g).sum()))
    if n <= max_norm or n == 0.0:
        return g
    return g * (max_norm / n)


def train_step(ck: Checkpoint, flat: np.ndarray, adam: Adam, tok, tgt, clip=5.0, masks=None):
    """One batch of train_model's loop: returns (new flat params, loss_sum)."""
    P = ck.unflat(flat)
    loss, G, _ = loss_and_grads(ck, P, tok, tgt, masks)
    g = ck.flat(G) / len(np.asarray(tok).reshape(-1, 7))
    return adam.apply(flat, clip_global_norm(g, clip)), loss
