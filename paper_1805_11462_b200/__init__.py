"""Python binding of the onmt B200 C-ABI (include/onmt.h) - argument marshalling only.

Every step of the translation path runs in `libonmt_b200.so` (hand-written sm_100a
CUDA); this module converts numpy / torch buffers to pointers and status codes to
exceptions.  There is no CPU fallback: importing works without a GPU (so the C-ABI
can be inspected), but every compute call needs the built library and a B200.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ONMT_LIB_PATH: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("ONMT_LIB_PATH") or os.path.join(_HERE, "libonmt_b200.so")

ONMT_OK = 0
STATUS = {0: "OK", -1: "INVALID_ARG", -2: "IO", -3: "FORMAT", -4: "UNSUPPORTED", -5: "ID_RANGE",
          -6: "EMPTY_SOURCE", -7: "CUDA", -8: "OOM"}
PREC = {"fp32": 0, "bf16": 1}
K_MAX = 16

EXPORTS = ["onmt_load_weights", "onmt_model_get_info", "onmt_set_stream", "onmt_encode", "onmt_translate",
           "onmt_translate_trace", "onmt_translate_dev", "onmt_set_option", "onmt_get_kernel_time",
           "onmt_kernel_launches", "onmt_free", "onmt_last_error", "onmt_test_gemm", "onmt_test_gen", "onmt_score",
           "onmt_translate_ex", "onmt_translate_copy", "onmt_graph_captures", "onmt_last_plan",
           "onmt_vp_handle", "onmt_vp_open", "onmt_vp_close"]


class OnmtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class _DecodeOpts(ctypes.Structure):
    """onmt_decode_opts (include/onmt.h)."""
    _fields_ = [("beam", ctypes.c_int32), ("max_len", ctypes.c_int32), ("length_penalty", ctypes.c_float),
                ("coverage_penalty", ctypes.c_float), ("n_best", ctypes.c_int32), ("replace_unk", ctypes.c_int32)]


class _Plan(ctypes.Structure):
    """onmt_plan_info (include/onmt.h)."""
    _fields_ = [(n, ctypes.c_int32) for n in ("rsplit", "fold", "gen_parts", "gate_tiles", "groups")]


class _Info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("layers", "emb", "hidden", "v_src", "v_tgt", "bidir", "attn_general", "precision")]


_lib = None


def lib():
    """Load libonmt_b200.so (built by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, F32, VP = ctypes.POINTER, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p
    L.onmt_load_weights.argtypes = [ctypes.c_char_p, I32, I32, P(VP)]
    L.onmt_model_get_info.argtypes = [VP, P(_Info)]
    L.onmt_set_stream.argtypes = [VP, VP]
    L.onmt_encode.argtypes = [VP, VP, VP, I32, I32, VP, VP, VP]
    L.onmt_translate.argtypes = [VP, VP, VP, I32, I32, I32, I32, F32, VP, VP, VP, VP, VP]
    L.onmt_translate_trace.argtypes = [VP, VP, VP, I32, I32, I32, I32, F32, VP, VP, VP, VP, VP, VP, VP, VP]
    L.onmt_translate_dev.argtypes = [VP, VP, VP, VP, I32, I32, I32, I32, F32, VP, VP, VP, VP, VP]
    L.onmt_set_option.argtypes = [VP, ctypes.c_char_p, I64]
    L.onmt_get_kernel_time.argtypes = [VP, ctypes.c_char_p, I32, P(ctypes.c_double), P(I64)]
    L.onmt_kernel_launches.argtypes = [VP, I32, P(I64)]
    L.onmt_graph_captures.argtypes = [VP, P(I64)]
    L.onmt_last_plan.argtypes = [VP, P(_Plan)]
    L.onmt_vp_handle.argtypes = [VP, I32, VP]
    L.onmt_vp_open.argtypes = [VP, I32, I32, VP]
    L.onmt_vp_close.argtypes = [VP]
    L.onmt_free.argtypes = [VP]
    L.onmt_free.restype = None
    L.onmt_last_error.restype = ctypes.c_char_p
    L.onmt_test_gemm.argtypes = [VP, VP, VP, I32, I32, I32, I32, VP]
    L.onmt_test_gen.argtypes = [VP, VP, I32, I32, VP, VP, VP]
    L.onmt_score.argtypes = [VP, VP, VP, I32, I32, VP, VP, I32, VP, VP]
    L.onmt_translate_ex.argtypes = [VP, VP, VP, I32, I32, P(_DecodeOpts), VP, VP, VP, VP, VP, VP]
    L.onmt_translate_copy.argtypes = [VP, VP, VP, VP, I32, I32, P(_DecodeOpts), VP, VP, VP, VP, VP]
    for n in EXPORTS:
        if n not in ("onmt_free", "onmt_last_error"):
            getattr(L, n).restype = ctypes.c_int
    _lib = L
    return L


def _check(st: int):
    if st != ONMT_OK:
        raise OnmtError(st, lib().onmt_last_error().decode())


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


class Model:
    """A device-resident model handle (onmt_load_weights / onmt_free)."""

    def __init__(self, mnmt_path: str, device: int = 0, precision: str = "bf16"):
        h = ctypes.c_void_p()
        _check(lib().onmt_load_weights(mnmt_path.encode(), device, PREC[precision], ctypes.byref(h)))
        self._h = h
        self.precision = precision
        inf = _Info()
        _check(lib().onmt_model_get_info(self._h, ctypes.byref(inf)))
        self.info = {n: getattr(inf, n) for n, _ in _Info._fields_}

    def close(self):
        if getattr(self, "_h", None):
            lib().onmt_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # --------------------------------------------------------------- options
    def set_option(self, name: str, value: int):
        _check(lib().onmt_set_option(self._h, name.encode(), int(value)))

    def set_stream(self, stream_ptr: int | None):
        _check(lib().onmt_set_stream(self._h, ctypes.c_void_p(stream_ptr) if stream_ptr else None))

    def kernel_time(self, name: str, reset: bool = True):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        _check(lib().onmt_get_kernel_time(self._h, name.encode(), int(reset), ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def launches(self, reset: bool = True) -> int:
        n = ctypes.c_int64()
        _check(lib().onmt_kernel_launches(self._h, int(reset), ctypes.byref(n)))
        return n.value

    def last_plan(self) -> Dict[str, int]:
        """How the last translate call ran (onmt_last_plan)."""
        p = _Plan()
        _check(lib().onmt_last_plan(self._h, ctypes.byref(p)))
        return {n: getattr(p, n) for n, _ in _Plan._fields_}

    # ---------------------------------------------- vocabulary-parallel generator (multi-GPU)
    def vp_handle(self, max_rows: int) -> bytes:
        """Allocate the exchange buffer for up to max_rows hypothesis rows; its IPC handle."""
        buf = ctypes.create_string_buffer(64)
        _check(lib().onmt_vp_handle(self._h, int(max_rows), buf))
        return buf.raw

    def vp_open(self, world: int, rank: int, handles: bytes | None):
        """Map every rank's exchange buffer (handles: world x 64 bytes in rank order)."""
        hb = ctypes.create_string_buffer(handles, len(handles)) if handles else None
        _check(lib().onmt_vp_open(self._h, int(world), int(rank), hb))

    def vp_close(self):
        _check(lib().onmt_vp_close(self._h))

    def graph_captures(self) -> int:
        n = ctypes.c_int64()
        _check(lib().onmt_graph_captures(self._h, ctypes.byref(n)))
        return n.value

    # --------------------------------------------------------------- compute
    def encode(self, ids, lens):
        ids, lens = _i32(ids), _i32(lens)
        B = len(lens)
        S = ids.shape[1] if ids.ndim == 2 else 1
        H, L = self.info["hidden"], self.info["layers"]
        mem = np.zeros((B, S, H), np.float32)
        h = np.zeros((L, B, H), np.float32)
        c = np.zeros((L, B, H), np.float32)
        _check(lib().onmt_encode(self._h, _ptr(ids), _ptr(lens), B, S, _ptr(mem), _ptr(h), _ptr(c)))
        return mem, h, c

    def translate_ex(self, ids, lens, beam: int, max_len: int, length_penalty: float = 0.0,
                     coverage_penalty: float = 0.0, n_best: int = 1, replace_unk: bool = False) -> Dict[str, np.ndarray]:
        """onmt_translate_ex: outputs shaped [B, n_best, ...] (final order)."""
        ids, lens = _i32(ids), _i32(lens)
        B = len(lens)
        S = ids.shape[1] if ids.ndim == 2 and B > 0 else 1
        n = max(n_best, 1)
        hyps = np.zeros((B, n, max_len), np.int32)
        olens = np.zeros((B, n), np.int32)
        scores = np.zeros((B, n), np.float32)
        raw = np.zeros((B, n), np.float32)
        tlogp = np.zeros((B, n, max_len), np.float32)
        unk = np.full((B, n, max_len), -1, np.int32) if replace_unk else None
        o = _DecodeOpts(beam, max_len, float(length_penalty), float(coverage_penalty), n_best, int(bool(replace_unk)))
        _check(lib().onmt_translate_ex(self._h, _ptr(ids), _ptr(lens), B, S, ctypes.byref(o), _ptr(hyps), _ptr(olens),
                                       _ptr(scores), _ptr(raw), _ptr(tlogp), _ptr(unk) if unk is not None else None))
        out = {"hyps": hyps, "lens": olens, "scores": scores, "raw": raw, "token_logp": tlogp}
        if unk is not None:
            out["unk_pos"] = unk
        return out

    def translate_copy(self, ids, lens, src_ext, beam: int, max_len: int,
                       length_penalty: float = 0.0) -> Dict[str, np.ndarray]:
        """onmt_translate_copy (copy / pointer-generator models): hyps over extended ids."""
        ids, lens, src_ext = _i32(ids), _i32(lens), _i32(src_ext)
        B = len(lens)
        S = ids.shape[1] if ids.ndim == 2 and B > 0 else 1
        hyps = np.zeros((B, max_len), np.int32)
        olens = np.zeros(B, np.int32)
        scores = np.zeros(B, np.float32)
        raw = np.zeros(B, np.float32)
        tlogp = np.zeros((B, max_len), np.float32)
        o = _DecodeOpts(beam, max_len, float(length_penalty), 0.0, 1, 0)
        _check(lib().onmt_translate_copy(self._h, _ptr(ids), _ptr(lens), _ptr(src_ext), B, S, ctypes.byref(o), _ptr(hyps),
                                         _ptr(olens), _ptr(scores), _ptr(raw), _ptr(tlogp)))
        return {"hyps": hyps, "lens": olens, "scores": scores, "raw": raw, "token_logp": tlogp}

    def translate(self, ids, lens, beam: int, max_len: int, length_penalty: float = 0.0,
                  trace: bool = False) -> Dict[str, np.ndarray]:
        ids, lens = _i32(ids), _i32(lens)
        B = len(lens)
        S = ids.shape[1] if ids.ndim == 2 and B > 0 else 1
        hyps = np.zeros((B, max_len), np.int32)
        olens = np.zeros(B, np.int32)
        scores = np.zeros(B, np.float32)
        raw = np.zeros(B, np.float32)
        tlogp = np.zeros((B, max_len), np.float32)
        out = {"hyps": hyps, "lens": olens, "scores": scores, "raw": raw, "token_logp": tlogp}
        if trace:
            n = max(max_len * B * beam, 1)
            sp = np.full(n, -1, np.int32)
            st = np.zeros(n, np.int32)
            ss = np.full(n, -np.inf, np.float64)
            _check(lib().onmt_translate_trace(self._h, _ptr(ids), _ptr(lens), B, S, beam, max_len,
                                              float(length_penalty), _ptr(hyps), _ptr(olens), _ptr(scores),
                                              _ptr(raw), _ptr(tlogp), _ptr(sp), _ptr(st), _ptr(ss)))
            shp = (max_len, B, beam)
            out.update(sel_parent=sp[:max_len * B * beam].reshape(shp), sel_token=st[:max_len * B * beam].reshape(shp),
                       sel_score=ss[:max_len * B * beam].reshape(shp))
        else:
            _check(lib().onmt_translate(self._h, _ptr(ids), _ptr(lens), B, S, beam, max_len,
                                        float(length_penalty), _ptr(hyps), _ptr(olens), _ptr(scores),
                                        _ptr(raw), _ptr(tlogp)))
        return out

    def score(self, ids, lens, tgt, tgt_lens) -> Dict[str, np.ndarray]:
        """Teacher-forced scoring: token_logp [B, T_max] (0 past each length) and nll [B]."""
        ids, lens, tgt, tgt_lens = _i32(ids), _i32(lens), _i32(tgt), _i32(tgt_lens)
        B = len(lens)
        S = ids.shape[1] if ids.ndim == 2 and B > 0 else 1
        T = tgt.shape[1] if tgt.ndim == 2 and B > 0 else 1
        tlogp = np.zeros((B, T), np.float32)
        nll = np.zeros(B, np.float64)
        _check(lib().onmt_score(self._h, _ptr(ids), _ptr(lens), B, S, _ptr(tgt), _ptr(tgt_lens), T, _ptr(tlogp),
                                _ptr(nll)))
        return {"token_logp": tlogp, "nll": nll}

    def translate_dev(self, ids_dev, lens_dev, beam: int, max_len: int, length_penalty: float,
                      out: Dict, lens_host=None):
        """Device-pointer variant: ids_dev/lens_dev/out[...] are CUDA torch tensors
        (int32 / float32); enqueued on the handle's stream, no synchronisation."""
        B, S = ids_dev.shape
        lh = _i32(lens_host) if lens_host is not None else None
        _check(lib().onmt_translate_dev(self._h, ids_dev.data_ptr(), lens_dev.data_ptr(), _ptr(lh), B, S, beam,
                                        max_len, float(length_penalty), out["hyps"].data_ptr(),
                                        out["lens"].data_ptr(), out["scores"].data_ptr(),
                                        out["raw"].data_ptr() if "raw" in out else None,
                                        out["token_logp"].data_ptr() if "token_logp" in out else None))

    def test_gemm(self, W: np.ndarray, X: np.ndarray, splits: int = 0) -> np.ndarray:
        W = np.ascontiguousarray(W, np.float32)
        X = np.ascontiguousarray(X, np.float32)
        M, K = W.shape
        N = X.shape[0]
        out = np.zeros((N, M), np.float32)
        _check(lib().onmt_test_gemm(self._h, _ptr(W), _ptr(X), M, N, K, splits, _ptr(out)))
        return out

    def test_gen(self, htilde: np.ndarray, k: int):
        h = np.ascontiguousarray(htilde, np.float32)
        R = h.shape[0]
        lse = np.zeros(R, np.float32)
        tz = np.zeros((R, k), np.float32)
        ti = np.zeros((R, k), np.int32)
        _check(lib().onmt_test_gen(self._h, _ptr(h), R, k, _ptr(lse), _ptr(tz), _ptr(ti)))
        return lse, tz, ti


def translate_corpus(model: Model, ids: np.ndarray, lens: np.ndarray, beam: int, max_len: int,
                     length_penalty: float = 0.0, batch: int = 30):
    """Translate a corpus in fixed-size batches (host API), concatenating results."""
    outs = []
    for s in range(0, len(lens), batch):
        L = lens[s:s + batch]
        S = int(L.max())
        outs.append(model.translate(ids[s:s + batch, :S], L, beam, max_len, length_penalty))
    return {k: np.concatenate([o[k] for o in outs]) for k in outs[0]} if outs else {}
