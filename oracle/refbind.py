"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libmtkref.so.

libmtkref.so is the UNMODIFIED reference (mtk, /root/reference/proj) compiled
from its own sources by oracle/Makefile plus oracle/ref_shim.cpp.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU arm may import this module;
the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libmtkref.so")

_ERRORS = {1: "DimensionError", 2: "NumericError", 3: "ContractError",
           4: "DataError", 5: "IoError", 6: "Error"}


class RefError(RuntimeError):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing -- run `make -C oracle`")
        L = C.CDLL(LIB_PATH)
        P, I64, U64, I = C.c_void_p, C.c_int64, C.c_uint64, C.c_int
        fp = C.POINTER(C.c_float)
        ip = C.POINTER(C.c_int32)
        lp = C.POINTER(C.c_int64)
        dp = C.POINTER(C.c_double)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_examples_create": (P, [I64, ip, lp, ip, lp]),
            "ref_examples_add_stream": (None, [P, I64, ip, lp]),
            "ref_examples_free": (None, [P]),
            "ref_batches_make": (P, [P, I64, U64, I]),
            "ref_batches_count": (I64, [P]),
            "ref_batch_shape": (None, [P, I64, lp]),
            "ref_batch_get": (None, [P, I64, ip, fp, ip, fp, lp]),
            "ref_batches_free": (None, [P]),
            "ref_model_create": (P, [C.c_char_p, U64]),
            "ref_model_free": (None, [P]),
            "ref_param_count": (I64, [P]),
            "ref_param_name": (C.c_char_p, [P, I64]),
            "ref_param_shape": (I, [P, C.c_char_p, lp]),
            "ref_param_get": (I, [P, C.c_char_p, fp]),
            "ref_param_set": (I, [P, C.c_char_p, fp]),
            "ref_grad_get": (I, [P, C.c_char_p, fp]),
            "ref_grad_set": (I, [P, C.c_char_p, fp]),
            "ref_state_get": (I, [P, I, C.c_char_p, fp]),
            "ref_adam_step": (I64, [P]),
            "ref_loss_grads": (I, [P, P, I64, U64, dp, fp]),
            "ref_forward_loss": (I, [P, P, I64, U64, dp]),
            "ref_adam_update": (I, [P, C.c_float]),
            "ref_train": (I, [P, P, I, I64, U64, I64, I64, C.c_float, I64, dp, lp]),
            "ref_train_async": (I, [P, P, I, I64, U64, I64, I64, C.c_float, I64, dp, lp]),
            "ref_parameter_total": (I64, [C.c_char_p]),
            "ref_beam_search": (I, [P, P, I64, I, C.c_double, I64, lp, lp, dp, ip, I64, I64]),
            "ref_score_batch": (I, [P, P, I64, dp]),
            "ref_train_ckpt": (I, [P, P, I, I64, U64, I64, I64, C.c_float, I64, C.c_char_p, I64,
                                   C.c_char_p, dp, lp]),
            "ref_save_model": (I, [P, C.c_char_p]),
            "ref_load_params": (I, [P, C.c_char_p]),
            "ref_save_checkpoint": (I, [P, C.c_char_p, I64, I64, I64]),
            "ref_load_checkpoint": (I, [P, C.c_char_p, lp]),
            "ref_matmul": (I, [I, lp, fp, I, lp, fp, I, lp, fp, I, I, C.c_float, C.c_float]),
            "ref_op_dot": (I, [I, lp, fp, I, lp, fp, I, I, fp, fp, fp, fp]),
            "ref_op_layernorm": (I, [I64, I64, fp, fp, fp, fp, fp, fp, fp, fp]),
            "ref_op_softmax": (I, [I, lp, fp, I, lp, fp, fp, fp, fp]),
            "ref_op_xent": (I, [I64, I64, I64, fp, ip, fp, dp, fp]),
            "ref_op_embed": (I, [I64, I64, fp, I64, I64, ip, fp, fp, fp]),
            "ref_op_gru": (I, [I64, I64, I64, I, fp, fp, fp, fp, fp, fp, fp, fp]),
            "ref_op_mha": (I, [I64, I64, I64, I64, I, fp, fp, fp, fp, I, fp, fp, fp, fp, fp]),
            "ref_op_program": (I, [C.c_char_p, I, ip, lp, C.POINTER(fp), fp, fp, I64, lp,
                                   C.POINTER(C.c_int), C.POINTER(fp)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc:
        raise RefError(_ERRORS.get(rc, "Error"), lib().ref_last_error().decode())


def _f(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _l(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _dims(a):
    return np.asarray(a.shape, dtype=np.int64)


# ------------------------------------------------------------------ data

class Examples:
    """vector<Example> with one source stream (data.h:38-44)."""

    def __init__(self, sources, targets, extra_streams=()):
        src = [np.asarray(s, dtype=np.int32) for s in sources]
        tgt = [np.asarray(t, dtype=np.int32) for t in targets]
        soff = np.zeros(len(src) + 1, dtype=np.int64)
        toff = np.zeros(len(tgt) + 1, dtype=np.int64)
        soff[1:] = np.cumsum([len(s) for s in src])
        toff[1:] = np.cumsum([len(t) for t in tgt])
        sflat = np.concatenate(src).astype(np.int32) if soff[-1] else np.zeros(1, np.int32)
        tflat = np.concatenate(tgt).astype(np.int32) if toff[-1] else np.zeros(1, np.int32)
        self.h = lib().ref_examples_create(len(src), _i(sflat), _l(soff), _i(tflat), _l(toff))
        self.n = len(src)
        for stream in extra_streams:  # further source streams (multi-source models)
            xs = [np.asarray(x, dtype=np.int32) for x in stream]
            xoff = np.zeros(len(xs) + 1, dtype=np.int64)
            xoff[1:] = np.cumsum([len(x) for x in xs])
            xflat = np.concatenate(xs).astype(np.int32)
            lib().ref_examples_add_stream(self.h, len(xs), _i(xflat), _l(xoff))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_examples_free(self.h)


def make_batches(examples: Examples, budget: int, seed: int, shuffle: bool = True):
    """makeBatches (data.cpp:226-282) -> list of dicts of numpy arrays."""
    L = lib()
    h = L.ref_batches_make(examples.h, budget, seed, int(shuffle))
    if not h:
        raise RefError("Error", L.ref_last_error().decode())
    out = []
    try:
        for i in range(L.ref_batches_count(h)):
            d = np.zeros(3, np.int64)
            L.ref_batch_shape(h, i, _l(d))
            rows, s, t = (int(x) for x in d)
            b = dict(src_ids=np.zeros((rows, s), np.int32), src_mask=np.zeros((rows, s), np.float32),
                     tgt_ids=np.zeros((rows, t), np.int32), tgt_mask=np.zeros((rows, t), np.float32),
                     sent_ids=np.zeros(rows, np.int64))
            L.ref_batch_get(h, i, _i(b["src_ids"]), _f(b["src_mask"]), _i(b["tgt_ids"]),
                            _f(b["tgt_mask"]), _l(b["sent_ids"]))
            out.append(b)
    finally:
        L.ref_batches_free(h)
    return out


class BatchSet:
    """Opaque vector<Batch> kept alive on the reference side."""

    def __init__(self, examples: Examples, budget: int, seed: int, shuffle: bool = True):
        L = lib()
        self.h = L.ref_batches_make(examples.h, budget, seed, int(shuffle))
        if not self.h:
            raise RefError("Error", L.ref_last_error().decode())
        self.count = L.ref_batches_count(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_batches_free(self.h)


# ----------------------------------------------------------------- model

class RefModel:
    """buildModel + a master ExpressionGraph with registered params, an Adam
    with adamDefaultsFor(config) and an AveragedParameters (train.h)."""

    def __init__(self, config_text: str, seed: int = 1):
        L = lib()
        self.h = L.ref_model_create(config_text.encode(), seed)
        if not self.h:
            raise RefError("Error", L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_model_free(self.h)

    def param_names(self):
        L = lib()
        return [L.ref_param_name(self.h, i).decode() for i in range(L.ref_param_count(self.h))]

    def shape(self, name):
        d = np.zeros(4, np.int64)
        r = lib().ref_param_shape(self.h, name.encode(), _l(d))
        return tuple(int(x) for x in d[:r])

    def param(self, name):
        out = np.zeros(self.shape(name), np.float32)
        _check(lib().ref_param_get(self.h, name.encode(), _f(out)))
        return out

    def set_param(self, name, value):
        v = f32(value).reshape(self.shape(name))
        _check(lib().ref_param_set(self.h, name.encode(), _f(v)))

    def grad(self, name):
        out = np.zeros(self.shape(name), np.float32)
        _check(lib().ref_grad_get(self.h, name.encode(), _f(out)))
        return out

    def set_grad(self, name, value):
        v = f32(value).reshape(self.shape(name))
        _check(lib().ref_grad_set(self.h, name.encode(), _f(v)))

    def state(self, which: str, name):
        out = np.zeros(self.shape(name), np.float32)
        _check(lib().ref_state_get(self.h, {"m": 0, "v": 1, "avg": 2}[which], name.encode(), _f(out)))
        return out

    def adam_step(self):
        return lib().ref_adam_step(self.h)

    def loss_grads(self, batches: BatchSet, i: int, graph_seed: int = 1):
        loss = C.c_double()
        tok = C.c_float()
        _check(lib().ref_loss_grads(self.h, batches.h, i, graph_seed, C.byref(loss), C.byref(tok)))
        return loss.value, tok.value

    def forward_loss(self, batches: BatchSet, i: int, graph_seed: int = 1):
        loss = C.c_double()
        _check(lib().ref_forward_loss(self.h, batches.h, i, graph_seed, C.byref(loss)))
        return loss.value

    def adam_update(self, lr: float):
        _check(lib().ref_adam_update(self.h, lr))

    def train(self, examples: Examples, workers=1, budget=256, seed=1, epochs=1,
              max_updates=-1, lr_base=3e-4, warmup=16000, async_=False):
        fl = C.c_double()
        up = C.c_int64()
        fn = lib().ref_train_async if async_ else lib().ref_train
        _check(fn(self.h, examples.h, workers, budget, seed, epochs, max_updates,
                  lr_base, warmup, C.byref(fl), C.byref(up)))
        return fl.value, up.value


    def train_ckpt(self, examples: Examples, workers=1, budget=256, seed=1, epochs=1,
                   max_updates=-1, lr_base=3e-4, warmup=16000, checkpoint_path="",
                   checkpoint_every=0, resume_from=""):
        """train.cpp:407-418 with checkpointing / resume."""
        fl = C.c_double()
        up = C.c_int64()
        _check(lib().ref_train_ckpt(self.h, examples.h, workers, budget, seed, epochs,
                                    max_updates, lr_base, warmup, checkpoint_path.encode(),
                                    checkpoint_every, resume_from.encode(), C.byref(fl),
                                    C.byref(up)))
        return fl.value, up.value

    def beam_search(self, batches: "BatchSet", i: int, rows: int, beam=5, alpha=0.6,
                    len_factor=3):
        """search.cpp beamSearch: per sentence [(tokens, score), ...] best first."""
        cap_h, cap_t = rows * beam * 2 + 8, rows * beam * 2 * 256
        counts = np.zeros(rows, np.int64)
        lens = np.zeros(cap_h, np.int64)
        scores = np.zeros(cap_h, np.float64)
        toks = np.zeros(cap_t, np.int32)
        _check(lib().ref_beam_search(self.h, batches.h, i, beam, alpha, len_factor, _l(counts),
                                     _l(lens), scores.ctypes.data_as(C.POINTER(C.c_double)),
                                     _i(toks), cap_h, cap_t))
        out, h, t = [], 0, 0
        for s in range(rows):
            hyps = []
            for _ in range(int(counts[s])):
                n = int(lens[h])
                hyps.append((toks[t:t + n].tolist(), float(scores[h])))
                t += n
                h += 1
            out.append(hyps)
        return out

    def score_batch(self, batches: "BatchSet", i: int, rows: int):
        out = np.zeros(rows, np.float64)
        _check(lib().ref_score_batch(self.h, batches.h, i, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def save_model(self, path: str):
        _check(lib().ref_save_model(self.h, path.encode()))

    def load_params(self, path: str):
        _check(lib().ref_load_params(self.h, path.encode()))

    def save_checkpoint(self, path: str, update: int, epoch: int, batch: int):
        _check(lib().ref_save_checkpoint(self.h, path.encode(), update, epoch, batch))

    def load_checkpoint(self, path: str):
        c = np.zeros(3, np.int64)
        _check(lib().ref_load_checkpoint(self.h, path.encode(), _l(c)))
        return tuple(int(x) for x in c)


def parameter_total(config_text: str) -> int:
    return int(lib().ref_parameter_total(config_text.encode()))


# -------------------------------------------------------------- op level

def matmul(a, b, trans_a=False, trans_b=False, alpha=1.0, beta=0.0, c=None):
    a, b = f32(a), f32(b)
    ra = a
    m = a.shape[-1] if trans_a else a.shape[-2]
    n = b.shape[-2] if trans_b else b.shape[-1]
    batch = max(a.shape[0] if a.ndim == 3 else 1, b.shape[0] if b.ndim == 3 else 1)
    shape = (batch, m, n) if (a.ndim == 3 or b.ndim == 3) else (m, n)
    c = np.zeros(shape, np.float32) if c is None else f32(c).copy()
    _check(lib().ref_matmul(ra.ndim, _l(_dims(ra)), _f(ra), b.ndim, _l(_dims(b)), _f(b),
                            c.ndim, _l(_dims(c)), _f(c), int(trans_a), int(trans_b), alpha, beta))
    return c


def op_dot(a, b, trans_a, trans_b, G):
    a, b, G = f32(a), f32(b), f32(G)
    out = np.zeros(G.shape, np.float32)
    ga, gb = np.zeros_like(a), np.zeros_like(b)
    _check(lib().ref_op_dot(
        a.ndim, _l(_dims(a)), _f(a), b.ndim, _l(_dims(b)), _f(b), int(trans_a), int(trans_b),
        _f(G), _f(out), _f(ga), _f(gb)))
    return out, ga, gb


def op_layernorm(x, gain, bias, G):
    x, gain, bias, G = f32(x), f32(gain), f32(bias), f32(G)
    rows, d = x.shape
    out, gx = np.zeros_like(x), np.zeros_like(x)
    gg, gb = np.zeros_like(gain), np.zeros_like(bias)
    _check(lib().ref_op_layernorm(rows, d, _f(x), _f(gain), _f(bias), _f(G), _f(out), _f(gx),
                                  _f(gg), _f(gb)))
    return out, gx, gg, gb


def op_softmax(x, mask, G):
    x, G = f32(x), f32(G)
    out, gx = np.zeros_like(x), np.zeros_like(x)
    if mask is None:
        _check(lib().ref_op_softmax(x.ndim, _l(_dims(x)), _f(x), 0, None, None, _f(G), _f(out), _f(gx)))
    else:
        m = f32(mask)
        _check(lib().ref_op_softmax(x.ndim, _l(_dims(x)), _f(x), m.ndim, _l(_dims(m)), _f(m),
                                    _f(G), _f(out), _f(gx)))
    return out, gx


def op_xent(logits, targets, mask):
    logits = f32(logits)
    b, t, V = logits.shape
    tg = np.ascontiguousarray(targets, dtype=np.int32)
    gl = np.zeros_like(logits)
    loss = C.c_double()
    m = None if mask is None else f32(mask)
    _check(lib().ref_op_xent(b, t, V, _f(logits), _i(tg), _f(m), C.byref(loss), _f(gl)))
    return loss.value, gl


def op_embed(table, ids, G):
    table, G = f32(table), f32(G)
    V, e = table.shape
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    rows, cols = ids.shape
    out = np.zeros((rows, cols, e), np.float32)
    gt = np.zeros_like(table)
    _check(lib().ref_op_embed(V, e, _f(table), rows, cols, _i(ids), _f(G), _f(out), _f(gt)))
    return out, gt


def op_mha(q, k, v, key_mask, causal, heads, G):
    """MultiHeadAttention with identity projections: the attention core."""
    q, k, v, G = f32(q), f32(k), f32(v), f32(G)
    b, tq, d = q.shape
    tk = k.shape[1]
    out = np.zeros_like(q)
    gq, gk, gv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    km = None if key_mask is None else f32(key_mask)
    _check(lib().ref_op_mha(b, tq, tk, d, heads, _f(q), _f(k), _f(v), _f(km), int(causal),
                            _f(G), _f(out), _f(gq), _f(gk), _f(gv)))
    return out, gq, gk, gv


def op_gru(h, x, packed_w, ln, G, e, d):
    h, G, packed_w = f32(h), f32(G), f32(packed_w)
    b = h.shape[0]
    xx = f32(x) if e > 0 else np.zeros(1, np.float32)
    out, gh = np.zeros_like(h), np.zeros_like(h)
    gx = np.zeros_like(xx)
    gw = np.zeros_like(packed_w)
    _check(lib().ref_op_gru(b, e, d, int(ln), _f(h), _f(xx), _f(packed_w), _f(G), _f(out),
                            _f(gh), _f(gx), _f(gw)))
    return out, gh, (gx if e > 0 else None), gw


def op_program(prog: str, inputs, G):
    """Run a stack program of reference graph ops (ref_shim.cpp ref_op_program)
    on parameters `inputs` with loss = sum(out * G).  Returns (out, [grads])."""
    ins = [f32(a) for a in inputs]
    ranks = np.asarray([a.ndim for a in ins], np.int32)
    dims = np.asarray([d for a in ins for d in a.shape] or [0], np.int64)
    ptrs = (C.POINTER(C.c_float) * max(len(ins), 1))(*[_f(a) for a in ins])
    grads = [np.zeros_like(a) for a in ins]
    gptrs = (C.POINTER(C.c_float) * max(len(ins), 1))(*[_f(a) for a in grads])
    Gf = f32(G).ravel()
    out = np.zeros(Gf.size, np.float32)
    odims = np.zeros(4, np.int64)
    orank = C.c_int()
    _check(lib().ref_op_program(prog.encode(), len(ins), _i(ranks), _l(dims), ptrs, _f(Gf),
                                _f(out), out.size, _l(odims), C.byref(orank), gptrs))
    shape = tuple(int(x) for x in odims[:orank.value])
    return out[:int(np.prod(shape))].reshape(shape), grads
