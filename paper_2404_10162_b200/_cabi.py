"""ctypes view of the engine's C-ABI (include/ks_b200.h).

This is the thin host binding used by tests and bench.py; the reference-style
API (``predict``, ``topk_metrics`` ...) lives in ``paper_2404_10162_b200.api``
and the C++ host library.  The shared library is built in-tree by
``__graft_entry__.build()``; importing without it raises, there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
import weakref
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libks_b200.so")

KS_OK = 0
STATUS_NAMES = {
    1: "ShapeError", 2: "ParameterError", 3: "IndexError", 4: "StateError",
    5: "ValidationError", 6: "CheckpointError", 7: "BeamExhaustedError", 8: "CudaError",
    9: "UnsupportedError",
}
PREC = {"f16x3": 0, "fp32": 1, "bf16": 2}
PRED_MASK, PRED_BUDGET, PRED_PRODUCT, PRED_DIVIDES = 1, 2, 3, 4


class KsError(RuntimeError):
    """Carries the C-ABI status code (one per reference exception class)."""

    def __init__(self, code: int, msg: str, field: str = ""):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.field = field


class KsPred(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("full_sequence_only", C.c_int32),
        ("allowed", C.POINTER(C.c_uint8)),
        ("n_terms", C.c_int32),
        ("term_pos", C.POINTER(C.c_int32)),
        ("term_w", C.POINTER(C.c_double)),
        ("term_field", C.POINTER(C.c_int32)),
        ("budget", C.c_double),
        ("scale", C.c_int64),
        ("limit", C.c_int64),
    ]


class KsModelDesc(C.Structure):
    _fields_ = [
        ("variant", C.c_int32),
        ("encoder_state_size", C.c_int32),
        ("pre_attention_size", C.c_int32),
        ("post_attention_size", C.c_int32),
        ("attention_dense_nodes", C.c_int32),
        ("num_positions", C.c_int32),
        ("input_sizes", C.POINTER(C.c_int32)),
        ("input_values", C.POINTER(C.c_int64)),
        ("vocab_sizes", C.POINTER(C.c_int32)),
        ("output_values", C.POINTER(C.c_int64)),
        ("num_tensors", C.c_int32),
        ("tensor_names", C.POINTER(C.c_char_p)),
        ("tensor_numel", C.POINTER(C.c_int32)),
        ("tensor_data", C.POINTER(C.POINTER(C.c_float))),
        ("decoder_cell_size", C.c_int32),
        ("num_conv_layers", C.c_int32),
        ("conv_layers", C.POINTER(C.c_int32)),
    ]


_lib = None

EXPORTS = [
    "ks_last_error", "ks_last_error_field", "ks_checkpoint_load", "ks_checkpoint_error_kind",
    "ks_checkpoint_free", "ks_checkpoint_header", "ks_checkpoint_num_tensors",
    "ks_checkpoint_tensor", "ks_engine_create", "ks_engine_create_from_checkpoint",
    "ks_engine_destroy", "ks_engine_num_positions", "ks_engine_vocab_size",
    "ks_engine_precision", "ks_engine_last_launch_count", "ks_engine_set_chunk",
    "ks_encode_problems", "ks_beam_search_batch", "ks_greedy_batch", "ks_beam_search_device",
    "ks_host_register", "ks_host_unregister",
    "ks_engine_profile_reset", "ks_engine_profile_gemm_ms", "ks_engine_profile_launches",
    "ks_engine_profile_launches_ex",
    "ks_beam_search_batch_hooked", "ks_topk_metrics_batch",
    "ks_trainer_create", "ks_trainer_create_from_checkpoint", "ks_trainer_destroy",
    "ks_trainer_num_params", "ks_trainer_num_ref_params", "ks_trainer_last_launch_count", "ks_trainer_loss_grads",
    "ks_trainer_apply", "ks_trainer_step", "ks_trainer_evaluate", "ks_trainer_export", "ks_trainer_import",
    "ks_trainer_to_reference_layout", "ks_synthetic_descriptors", "ks_engine_synthetic_descriptors", "ks_forward_batch",
    "ks_device_count", "ks_engine_group_create", "ks_engine_group_create_from_checkpoint", "ks_engine_group_destroy",
    "ks_engine_group_size", "ks_engine_group_engine", "ks_group_beam_search_batch", "ks_group_greedy_batch",
    "ks_group_forward_batch", "ks_group_topk_metrics_batch", "ks_topk_metrics_multi",
    "ks_group_topk_metrics_multi", "ks_gemm_f16x3",
]


def pin_results(out):
    """Page-lock the result arrays of a beam() call for their lifetime, so later
    calls reusing them (`out=`) receive the device-to-host copy directly.
    Registration costs tens of ms for a 65k-config result set: worth it only for a
    long-running loop over the same buffers."""
    for a in out.values():
        if isinstance(a, np.ndarray):
            _pin(a)
    return out


def _pin(a):
    """Page-lock a numpy array for the array's lifetime (ks_host_register)."""
    L = lib()
    ptr = a.ctypes.data
    if L.ks_host_register(C.c_void_p(ptr), a.nbytes) == 0:
        weakref.finalize(a, L.ks_host_unregister, C.c_void_p(ptr))


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def lib():
    """Loads libks_b200.so (raises if the extension was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(the engine has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    L.ks_last_error.restype = C.c_char_p
    L.ks_last_error_field.restype = C.c_char_p
    L.ks_checkpoint_load.argtypes = [C.c_char_p, P(vp)]
    L.ks_host_register.argtypes = [vp, C.c_int64]
    L.ks_host_unregister.argtypes = [vp]
    L.ks_gemm_f16x3.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, C.c_float, vp, i64, vp]
    L.ks_checkpoint_error_kind.restype = i32
    L.ks_checkpoint_free.argtypes = [vp]
    L.ks_checkpoint_header.argtypes = [vp, C.c_char_p]
    L.ks_checkpoint_header.restype = C.c_char_p
    L.ks_checkpoint_num_tensors.argtypes = [vp]
    L.ks_checkpoint_tensor.argtypes = [vp, i32, P(C.c_char_p), P(i32), P(i32), P(P(C.c_float))]
    L.ks_engine_create.argtypes = [P(KsModelDesc), i32, i32, P(vp)]
    L.ks_engine_create_from_checkpoint.argtypes = [C.c_char_p, i32, i32, P(vp)]
    L.ks_engine_destroy.argtypes = [vp]
    L.ks_engine_num_positions.argtypes = [vp]
    L.ks_engine_vocab_size.argtypes = [vp, i32]
    L.ks_engine_precision.argtypes = [vp]
    L.ks_engine_last_launch_count.argtypes = [vp]
    L.ks_engine_last_launch_count.restype = i64
    L.ks_engine_set_chunk.argtypes = [vp, i64]
    L.ks_encode_problems.argtypes = [vp, P(i64), i64, i32, P(i32), P(i64)]
    L.ks_beam_search_batch.argtypes = [vp, P(i32), P(i64), i64, i32, P(KsPred), i32, P(i32),
                                       P(dbl), P(i32), P(i32), P(i32), P(i32)]
    L.ks_greedy_batch.argtypes = [vp, P(i32), i64, P(i32)]
    L.ks_beam_search_device.argtypes = [vp, vp, vp, i64, i32, P(KsPred), i32, vp, vp, vp, vp, vp,
                                        vp, vp]
    L.ks_engine_profile_reset.argtypes = [vp, i32]
    L.ks_engine_profile_gemm_ms.argtypes = [vp, P(i64), P(dbl)]
    L.ks_engine_profile_gemm_ms.restype = dbl
    L.ks_engine_profile_launches.argtypes = [vp, i64, P(dbl), P(dbl)]
    L.ks_engine_profile_launches.restype = i64
    L.ks_engine_profile_launches_ex.argtypes = [vp, i64, P(dbl), P(dbl), P(dbl)]
    L.ks_engine_profile_launches_ex.restype = i64
    L.ks_trainer_create.argtypes = [P(KsModelDesc), dbl, dbl, i32, P(vp)]
    L.ks_trainer_create_from_checkpoint.argtypes = [C.c_char_p, i32, P(vp)]
    L.ks_trainer_destroy.argtypes = [vp]
    L.ks_trainer_num_params.argtypes = [vp]
    L.ks_trainer_num_params.restype = i64
    L.ks_trainer_num_ref_params.argtypes = [vp]
    L.ks_trainer_num_ref_params.restype = i64
    L.ks_trainer_last_launch_count.argtypes = [vp]
    L.ks_trainer_last_launch_count.restype = i64
    L.ks_trainer_loss_grads.argtypes = [vp, vp, vp, vp, i64, i64, C.c_uint64, vp, i32, vp, vp, vp]
    L.ks_trainer_apply.argtypes = [vp, vp, i64, dbl, dbl, vp]
    L.ks_trainer_step.argtypes = [vp, P(i32), P(i32), P(i64), i64, i64, C.c_uint64, dbl, dbl,
                                  P(dbl), P(i64)]
    L.ks_trainer_evaluate.argtypes = [vp, P(i32), P(i32), i64, P(dbl), P(i64)]
    L.ks_trainer_export.argtypes = [vp, P(C.c_float)]
    L.ks_trainer_import.argtypes = [vp, P(C.c_float)]
    L.ks_trainer_to_reference_layout.argtypes = [vp, P(C.c_float), P(C.c_float)]
    L.ks_engine_group_create_from_checkpoint.argtypes = [C.c_char_p, P(i32), i32, i32, P(vp)]
    L.ks_engine_group_destroy.argtypes = [vp]
    L.ks_engine_group_size.argtypes = [vp]
    L.ks_engine_group_engine.argtypes = [vp, i32]
    L.ks_engine_group_engine.restype = vp
    L.ks_group_beam_search_batch.argtypes = [vp, P(i32), P(i64), i64, i32, P(KsPred), i32, vp, vp, P(i32),
                                             P(dbl), P(i32), P(i32), P(i32), P(i32)]
    L.ks_group_greedy_batch.argtypes = [vp, P(i32), i64, P(i32)]
    L.ks_forward_batch.argtypes = [vp, P(i32), P(i32), i64, P(dbl), P(i32), P(dbl)]
    L.ks_synthetic_descriptors.argtypes = [P(i32), P(i64), C.c_uint64, i64, i64, P(i64)]
    L.ks_engine_synthetic_descriptors.argtypes = [vp, C.c_uint64, i64, i64, P(i64)]
    _lib = L
    return L


def gemm_f16x3(A, B, C=None, ta=False, tb=False, beta=0.0, stream=None):
    """ks_gemm_f16x3 on CUDA fp32 torch tensors (row-major, unit column stride):
    C = op(A) op(B) + beta C with op = transpose when ta / tb; returns C."""
    import torch
    M, K = (A.shape[1], A.shape[0]) if ta else (A.shape[0], A.shape[1])
    N = B.shape[0] if tb else B.shape[1]
    if (B.shape[1] if tb else B.shape[0]) != K:
        raise ValueError("inner dimensions differ")
    if C is None:
        C = torch.zeros((M, N), dtype=torch.float32, device=A.device)
    for t in (A, B, C):
        if t.dtype != torch.float32 or not t.is_cuda or t.stride(1) != 1:
            raise ValueError("CUDA fp32 tensors with unit column stride expected")
    s = torch.cuda.current_stream().cuda_stream if stream is None else stream
    check(lib().ks_gemm_f16x3(int(ta), int(tb), M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                              float(beta), C.data_ptr(), C.stride(0), s))
    return C


def synthetic_descriptors(input_values, count, seed=2404, start=0):
    """ks_synthetic_descriptors over a vocabulary given as 7 lists of field
    values: configs start..start+count-1, each from Rng::derive(seed, i)."""
    sizes = np.array([len(v) for v in input_values], np.int32)
    vals = np.concatenate([np.asarray(v, np.int64) for v in input_values])
    out = np.empty((count, 7), np.int64)
    check(lib().ks_synthetic_descriptors(_p(sizes, C.c_int32), _p(vals, C.c_int64), seed, start, count,
                                         _p(out, C.c_int64)))
    return out


def check(code: int):
    if code != KS_OK:
        L = lib()
        raise KsError(code, L.ks_last_error().decode(), L.ks_last_error_field().decode())


def pack_preds(preds):
    """preds: list of dicts {kind, full, allowed | term_pos/term_w/term_field, budget, scale, limit}."""
    arr = (KsPred * max(1, len(preds)))()
    keep = []
    for i, d in enumerate(preds):
        a = arr[i]
        a.kind = d["kind"]
        a.full_sequence_only = int(bool(d.get("full", False)))
        for key, ct in (("allowed", C.c_uint8), ("term_pos", C.c_int32), ("term_w", C.c_double),
                        ("term_field", C.c_int32)):
            if key in d and d[key] is not None:
                v = np.ascontiguousarray(d[key])
                keep.append(v)
                setattr(a, key, _p(v, ct))
        if "term_pos" in d:
            a.n_terms = len(d["term_pos"])
        a.budget = float(d.get("budget", 0.0))
        a.scale = int(d.get("scale", 1))
        a.limit = int(d.get("limit", 0))
    return arr, keep


class Engine:
    """One engine per GPU; immutable weights, reusable workspace."""

    def __init__(self, checkpoint: str, device: int = 0, precision: str = "f16x3"):
        L = lib()
        h = C.c_void_p()
        check(L.ks_engine_create_from_checkpoint(checkpoint.encode(), device, PREC[precision],
                                                 C.byref(h)))
        self._h = h
        self._destroy = L.ks_engine_destroy  # bound now: module globals may be gone at shutdown
        self.T = L.ks_engine_num_positions(h)
        self.vsizes = [L.ks_engine_vocab_size(h, p) for p in range(self.T)]
        self.precision = precision

    def close(self):
        if getattr(self, "_h", None):
            self._destroy(self._h)
            self._h = None

    __del__ = close

    def set_chunk(self, n: int):
        check(lib().ks_engine_set_chunk(self._h, n))

    def launches(self) -> int:
        return lib().ks_engine_last_launch_count(self._h)

    def synthetic(self, count, seed=2404, start=0):
        """Synthetic descriptors over the model's input vocabulary (ks_engine_synthetic_descriptors)."""
        out = np.empty((count, 7), np.int64)
        check(lib().ks_engine_synthetic_descriptors(self._h, seed, start, count, _p(out, C.c_int64)))
        return out

    def encode(self, desc, allow_nearest=False):
        desc = np.ascontiguousarray(desc, np.int64).reshape(-1, 7)
        tok = np.zeros(desc.shape, np.int32)
        bad = C.c_int64(-1)
        check(lib().ks_encode_problems(self._h, _p(desc, C.c_int64), len(desc), int(allow_nearest),
                                       _p(tok, C.c_int32), C.byref(bad)))
        return tok

    def beam(self, tok, k, desc=None, preds=(), out=None):
        """ks_beam_search_batch.  `out` (optional) is a dict of caller-owned result
        arrays from a previous call with the same B and k, reused in place."""
        tok = np.ascontiguousarray(tok, np.int32).reshape(-1, 7)
        B = len(tok)
        d = None if desc is None else np.ascontiguousarray(desc, np.int64).reshape(-1, 7)
        if out is not None and out["tokens"].shape == (B, k, self.T):
            out_tok, out_lp, cnt = out["tokens"], out["log_prob"], out["count"]
            st, fp, fs = out["status"], out["fail_pred"], out["fail_step"]

        else:
            out_tok = np.empty((B, k, self.T), np.int32)
            out_lp = np.empty((B, k), np.float64)
            cnt = np.empty(B, np.int32)
            st = np.empty(B, np.int32)
            fp = np.empty(B, np.int32)
            fs = np.empty(B, np.int32)
        arr, keep = pack_preds(list(preds))
        check(lib().ks_beam_search_batch(self._h, _p(tok, C.c_int32), _p(d, C.c_int64), B, k, arr,
                                         len(preds), _p(out_tok, C.c_int32), _p(out_lp, C.c_double),
                                         _p(cnt, C.c_int32), _p(st, C.c_int32), _p(fp, C.c_int32),
                                         _p(fs, C.c_int32)))
        return {"tokens": out_tok, "log_prob": out_lp, "count": cnt, "status": st,
                "fail_pred": fp, "fail_step": fs}

    def greedy(self, tok):
        tok = np.ascontiguousarray(tok, np.int32).reshape(-1, 7)
        out = np.empty((len(tok), self.T), np.int32)
        check(lib().ks_greedy_batch(self._h, _p(tok, C.c_int32), len(tok), _p(out, C.c_int32)))
        return out

    def forward(self, tok, teacher=None):
        """ks_forward_batch: per-position distributions (list of B x V_p arrays), the
        fed-back tokens (B x T) and the sequence scores (B)."""
        tok = np.ascontiguousarray(tok, np.int32).reshape(-1, 7)
        B = len(tok)
        t = None if teacher is None else np.ascontiguousarray(teacher, np.int32).reshape(B, self.T)
        sv = sum(self.vsizes)
        dist = np.empty((B, sv), np.float64)
        fed = np.empty((B, self.T), np.int32)
        score = np.empty(B, np.float64)
        check(lib().ks_forward_batch(self._h, _p(tok, C.c_int32), _p(t, C.c_int32), B, _p(dist, C.c_double),
                                     _p(fed, C.c_int32), _p(score, C.c_double)))
        offs = np.cumsum([0] + self.vsizes)
        return [dist[:, offs[p]:offs[p + 1]] for p in range(self.T)], fed, score

    def beam_device(self, d_tok, d_desc, B, k, preds, d_out, stream=0):
        """All buffers are device pointers (ints); d_out = dict of pointers."""
        arr, keep = pack_preds(list(preds))
        check(lib().ks_beam_search_device(self._h, d_tok, d_desc, B, k, arr, len(preds),
                                          d_out["tokens"], d_out["log_prob"], d_out["count"],
                                          d_out.get("status"), d_out.get("fail_pred"),
                                          d_out.get("fail_step"), stream))

    def profile_reset(self, enable=True):
        lib().ks_engine_profile_reset(self._h, int(enable))

    def profile_launches(self):
        """Per gate-GEMM launch of the last profiled call: (ms, useful FLOPs by the
        reference formula, FLOPs issued to the tensor pipe)."""
        n = lib().ks_engine_profile_launches(self._h, 0, None, None)
        ms, fl, ex = np.zeros(n), np.zeros(n), np.zeros(n)
        lib().ks_engine_profile_launches_ex(self._h, n, _p(ms, C.c_double), _p(fl, C.c_double),
                                            _p(ex, C.c_double))
        return ms, fl, ex

    def profile(self):
        n = C.c_int64(0)
        useful = C.c_double(0.0)
        ms = lib().ks_engine_profile_gemm_ms(self._h, C.byref(n), C.byref(useful))
        return ms, n.value, useful.value


class EngineGroup:
    """One engine per listed device (None: every visible GPU); batches are
    sharded contiguously across them (ks_group_*), results in config order."""

    def __init__(self, checkpoint: str, devices=None, precision: str = "f16x3"):
        L = lib()
        h = C.c_void_p()
        devs = None if devices is None else np.ascontiguousarray(devices, np.int32)
        check(L.ks_engine_group_create_from_checkpoint(checkpoint.encode(), _p(devs, C.c_int32),
                                                       0 if devs is None else len(devs), PREC[precision],
                                                       C.byref(h)))
        self._h = h
        self._destroy = L.ks_engine_group_destroy
        self.size = L.ks_engine_group_size(h)
        self.T = L.ks_engine_num_positions(L.ks_engine_group_engine(h, 0))

    def close(self):
        if getattr(self, "_h", None):
            self._destroy(self._h)
            self._h = None

    __del__ = close

    def beam(self, tok, k, desc=None, preds=()):
        tok = np.ascontiguousarray(tok, np.int32).reshape(-1, 7)
        B = len(tok)
        d = None if desc is None else np.ascontiguousarray(desc, np.int64).reshape(-1, 7)
        out_tok = np.empty((B, k, self.T), np.int32)
        out_lp = np.empty((B, k), np.float64)
        cnt, st, fp, fs = (np.empty(B, np.int32) for _ in range(4))
        arr, keep = pack_preds(list(preds))
        check(lib().ks_group_beam_search_batch(self._h, _p(tok, C.c_int32), _p(d, C.c_int64), B, k, arr, len(preds),
                                               None, None, _p(out_tok, C.c_int32), _p(out_lp, C.c_double),
                                               _p(cnt, C.c_int32), _p(st, C.c_int32), _p(fp, C.c_int32),
                                               _p(fs, C.c_int32)))
        return {"tokens": out_tok, "log_prob": out_lp, "count": cnt, "status": st, "fail_pred": fp,
                "fail_step": fs}


class Trainer:
    """Teacher-forced training on one GPU (BASELINE config 4): the C-ABI
    ks_trainer_* (train_model's batch body, proj/src/models.cpp:905-947).
    Device-buffer calls take raw device pointers (ints) and a cudaStream_t."""

    def __init__(self, checkpoint: str, device: int = 0):
        L = lib()
        h = C.c_void_p()
        check(L.ks_trainer_create_from_checkpoint(checkpoint.encode(), device, C.byref(h)))
        self._h = h
        self._destroy = L.ks_trainer_destroy
        self.num_params = L.ks_trainer_num_params(h)          # train-layout buffers (grads)
        self.num_ref_params = L.ks_trainer_num_ref_params(h)  # reference order (export/import)

    def close(self):
        if getattr(self, "_h", None):
            self._destroy(self._h)
            self._h = None

    __del__ = close

    def launches(self) -> int:
        return lib().ks_trainer_last_launch_count(self._h)

    def loss_grads_device(self, d_tok, d_tgt, d_idx, B, dropout_epoch, seed, d_grads, accumulate,
                          d_loss, d_match, stream=0):
        check(lib().ks_trainer_loss_grads(self._h, d_tok, d_tgt, d_idx, B, dropout_epoch, seed, d_grads,
                                          int(accumulate), d_loss, d_match, stream))

    def apply_device(self, d_grads, batch, lr, clip=5.0, stream=0):
        check(lib().ks_trainer_apply(self._h, d_grads, batch, lr, clip, stream))

    def step(self, tok, tgt, idx=None, epoch=-1, seed=0, lr=1e-3, clip=5.0):
        """Host-buffer step: returns (loss_sum, matches)."""
        tok = np.ascontiguousarray(tok, np.int32).reshape(-1, 7)
        tgt = np.ascontiguousarray(tgt, np.int32).reshape(len(tok), -1)
        ix = None if idx is None else np.ascontiguousarray(idx, np.int64)
        loss = C.c_double()
        m = C.c_int64()
        check(lib().ks_trainer_step(self._h, _p(tok, C.c_int32), _p(tgt, C.c_int32), _p(ix, C.c_int64),
                                    len(tok), epoch, seed, lr, clip, C.byref(loss), C.byref(m)))
        return loss.value, m.value

    def export(self) -> np.ndarray:
        out = np.empty(self.num_ref_params, np.float32)
        check(lib().ks_trainer_export(self._h, _p(out, C.c_float)))
        return out

    def import_(self, flat_ref):
        v = np.ascontiguousarray(flat_ref, np.float32)
        check(lib().ks_trainer_import(self._h, _p(v, C.c_float)))

    def to_reference_layout(self, train_flat) -> np.ndarray:
        v = np.ascontiguousarray(train_flat, np.float32)
        out = np.empty(self.num_ref_params, np.float32)
        check(lib().ks_trainer_to_reference_layout(self._h, _p(v, C.c_float), _p(out, C.c_float)))
        return out
