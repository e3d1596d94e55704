"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

ctypes bindings for
  * liboracle.so           : the plain-C restatement (oracle/absp_oracle.c)
  * _ref/libabsparse_ref.so: the unmodified reference core + C shim (oracle/ref_shim.cpp)
and the batch / GQA layering of SURVEY.md Appendix A on top of the per-sequence
reference functions.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_ORACLE = HERE / "liboracle.so"
LIB_REF = HERE / "_ref" / "libabsparse_ref.so"

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def build_oracle(ref: bool = False) -> None:
    """Compile the C restatement (and the reference core when its sources exist)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if ref and Path("/root/reference/proj/src").is_dir():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


_oracle = None
_ref = None


def lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not LIB_ORACLE.exists():
            build_oracle()
        L = C.CDLL(str(LIB_ORACLE))
        L.absp_oracle_offsets.argtypes = [_sz, _u32p, _sz, _u64p]
        L.absp_oracle_centroids.argtypes = [_u16p, _sz, _u32p, _sz, _sz, _sz, _sz, _u32p, C.c_int,
                                            _f32p, C.c_void_p]
        L.absp_oracle_quantize.argtypes = [_f32p, _u64p, _sz, _sz, C.c_int, C.c_int, _u8p, _f32p, _f32p]
        L.absp_oracle_scores_quant.argtypes = [_f32p, _u8p, C.c_void_p, _f32p, _f32p, C.c_void_p,
                                               C.c_void_p, _u64p, _sz, _sz, C.c_int, C.c_int, C.c_int, _f32p]
        L.absp_oracle_scores_f32.argtypes = [_f32p, _f32p, C.c_void_p, _u64p, _sz, _sz, C.c_int, _f32p]
        L.absp_oracle_select.argtypes = [_f32p, _u64p, _u32p, _sz, _sz, _sz, _u32p, _sz, _u32p, C.c_void_p]
        L.absp_oracle_attend.argtypes = [_f32p, _u16p, _u16p, _sz, _u32p, _sz, _sz, _sz, _sz, _u32p,
                                         _u32p, _sz, _u32p, _f32p]
        L.absp_oracle_full_attention.argtypes = [_f32p, _u16p, _u16p, _sz, _u32p, _sz, _sz, _sz, _sz, _f32p]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return LIB_REF.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not LIB_REF.exists():
            raise FileNotFoundError(f"{LIB_REF} not built (make -C oracle ref, needs /root/reference)")
        L = C.CDLL(str(LIB_REF))
        L.ref_last_error.restype = C.c_char_p
        L.ref_seq_create.argtypes = [_sz, _sz, _sz, _sz, _sz, _f32p, _f32p, C.POINTER(_sz), C.c_int,
                                     C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_seq_destroy.argtypes = [C.c_void_p]
        L.ref_seq_total_centroids.argtypes = [C.c_void_p]
        L.ref_seq_total_centroids.restype = _sz
        L.ref_seq_offsets.argtypes = [C.c_void_p, _u64p]
        L.ref_seq_store.argtypes = [C.c_void_p] + [C.c_void_p] * 8
        L.ref_seq_estimate.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ref_seq_estimate_naive.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ref_seq_select.argtypes = [C.c_void_p, _f32p, _sz, _u32p, _sz, _u32p, _u32p]
        L.ref_seq_select_naive.argtypes = [C.c_void_p, _f32p, _sz, _u32p, _sz, _u32p]
        L.ref_seq_attend.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ref_seq_full_attention.argtypes = [C.c_void_p, _f32p, _f32p]
        L.ref_seq_full_attention_w.argtypes = [C.c_void_p, _f32p, _f32p,
                                               np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]
        L.ref_seq_decode_gqa.argtypes = [C.c_void_p, _f32p, _sz, _sz, _f32p]
        L.ref_engine_create.argtypes = [_sz, _sz, _sz, C.POINTER(_sz), _sz, _sz, C.c_int, C.c_int,
                                        C.c_int, C.POINTER(_sz), _sz, C.POINTER(C.c_void_p)]
        L.ref_engine_destroy.argtypes = [C.c_void_p]
        L.ref_engine_prefill.argtypes = [C.c_void_p, _f32p, _f32p, _sz, _sz]
        L.ref_engine_step.argtypes = [C.c_void_p, _f32p, _f32p, _f32p, _f32p, C.c_void_p, _sz,
                                      C.c_void_p, C.POINTER(C.c_int)]
        L.ref_engine_store.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.POINTER(_sz)]
        _f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        L.ref_save_trace.argtypes = [C.c_char_p, _sz, _sz, _sz, C.c_uint64, _f32p, _f32p, _f32p]
        L.ref_load_trace.argtypes = [C.c_char_p, _u64p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_profile_sensitivity.argtypes = [_sz, _sz, _sz, C.POINTER(_sz), _sz, _sz, C.c_int, C.c_int, C.c_int,
                                              _sz, _sz, _f32p, _f32p, _f32p, _f64p]
        L.ref_transfer_check.argtypes = [_sz, _sz, _sz, C.POINTER(_sz), _sz, _sz, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(_sz), _sz, _sz, _f32p, _f32p, _f32p, _f64p]
        L.ref_write_recall_csv.argtypes = [C.c_char_p, _sz, C.POINTER(_sz), _sz, _f64p, C.c_char_p]
        L.ref_write_min_block_csv.argtypes = [C.c_char_p, C.POINTER(_sz), _sz, C.c_char_p]
        L.ref_assign_block_sizes.argtypes = [_sz, C.POINTER(_sz), _sz, _f64p, C.c_double, C.POINTER(_sz)]
        L.ref_config_validate.argtypes = [_sz, _sz, _sz, C.POINTER(_sz), _sz, _sz, C.c_int]
        L.ref_generate_synthetic.argtypes = [_sz, _sz, _sz, C.POINTER(C.c_int), C.POINTER(_sz),
                                             C.POINTER(_sz), C.c_double, C.c_uint64, _sz, _f32p,
                                             _f32p, _f32p]
        _ref = L
    return _ref


class RefError(Exception):
    """Reference exception, `kind` in {invalid_argument, out_of_range, runtime_error, logic_error}."""

    KINDS = {1: "invalid_argument", 2: "out_of_range", 3: "runtime_error", 4: "logic_error", 9: "other"}

    def __init__(self, code: int, msg: str):
        super().__init__(f"{self.KINDS.get(code, code)}: {msg}")
        self.kind = self.KINDS.get(code, "other")


def _rcheck(rc: int) -> None:
    if rc != 0:
        raise RefError(rc, ref().ref_last_error().decode())


def bf16_to_f32(x: np.ndarray) -> np.ndarray:
    return (x.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = u + 0x7FFF + ((u >> 16) & 1)
    return (u >> 16).astype(np.uint16)


# ---------------------------------------------------------------------------
# Per-sequence C restatement on the paged bf16 layout
# ---------------------------------------------------------------------------
class OracleSeq:
    """One sequence of a paged layer, evaluated by the C restatement.

    k_pool/v_pool: uint16 [H][pool_pages][P][d]; page_table: uint32 [pages of this seq].
    """

    def __init__(self, k_pool, v_pool, page_table, n, H, d, P, block_sizes, method=0, bits=4, mode=1):
        self.k_pool = np.ascontiguousarray(k_pool, dtype=np.uint16)
        self.v_pool = np.ascontiguousarray(v_pool, dtype=np.uint16)
        self.pool_pages = self.k_pool.shape[1]
        self.page_table = np.ascontiguousarray(page_table, dtype=np.uint32)
        self.n, self.H, self.d, self.P = int(n), int(H), int(d), int(P)
        self.block_sizes = np.ascontiguousarray(block_sizes, dtype=np.uint32)
        self.method, self.bits, self.mode = method, bits, mode
        L = lib()
        self.offsets = np.zeros(self.H + 1, np.uint64)
        L.absp_oracle_offsets(self.n, self.block_sizes, self.H, self.offsets)
        total = int(self.offsets[-1])
        self.values = np.zeros((total, self.d), np.float32)
        self.values_min = np.zeros((total, self.d), np.float32) if method == 1 else None
        rc = L.absp_oracle_centroids(self.k_pool, self.pool_pages, self.page_table, self.n, self.H, self.d,
                                     self.P, self.block_sizes, method, self.values,
                                     self.values_min.ctypes.data if method == 1 else None)
        if rc:
            raise ValueError("compute_block_centroids: cache is empty")
        self.codes = self.codes_min = self.scales = self.zps = self.scales_min = self.zps_min = None
        if bits:
            self.codes, self.scales, self.zps = self._quant(self.values)
            if method == 1:
                self.codes_min, self.scales_min, self.zps_min = self._quant(self.values_min)

    def _quant(self, vals):
        codes = np.zeros(vals.shape, np.uint8)
        sc = np.zeros((self.H, self.d), np.float32)
        zp = np.zeros((self.H, self.d), np.float32)
        rc = lib().absp_oracle_quantize(vals, self.offsets, self.H, self.d, self.bits, self.mode, codes, sc, zp)
        if rc:
            raise ValueError("quantize_store failed")
        return codes, sc, zp

    @property
    def total(self) -> int:
        return int(self.offsets[-1])

    def scores(self, q: np.ndarray) -> np.ndarray:
        """q: fp32 [H][d] (the KV-head queries)."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        out = np.zeros(self.total, np.float32)
        L = lib()
        if self.bits:
            ptr = lambda a: a.ctypes.data if a is not None else None
            L.absp_oracle_scores_quant(q, self.codes, ptr(self.codes_min), self.scales, self.zps,
                                       ptr(self.scales_min), ptr(self.zps_min), self.offsets, self.H,
                                       self.d, self.bits, self.mode, self.method, out)
        else:
            L.absp_oracle_scores_f32(q, self.values,
                                     self.values_min.ctypes.data if self.values_min is not None else None,
                                     self.offsets, self.H, self.d, self.method, out)
        return out

    def select(self, scores: np.ndarray, token_budget: int, max_k: int | None = None):
        if max_k is None:
            max_k = max(int(np.ceil(token_budget / b)) for b in self.block_sizes)
            max_k = max(max_k, 1)
        blocks = np.zeros((self.H, max_k), np.uint32)
        counts = np.zeros(self.H, np.uint32)
        rc = lib().absp_oracle_select(np.ascontiguousarray(scores, np.float32), self.offsets, self.block_sizes,
                                      self.H, self.n, token_budget, blocks, max_k, counts, None)
        if rc:
            raise ValueError("select_topk: invalid arguments")
        return [blocks[h, : counts[h]].copy() for h in range(self.H)]

    def attend(self, q: np.ndarray, selection) -> np.ndarray:
        max_k = max(len(s) for s in selection)
        blocks = np.zeros((self.H, max_k), np.uint32)
        counts = np.zeros(self.H, np.uint32)
        for h, s in enumerate(selection):
            blocks[h, : len(s)] = s
            counts[h] = len(s)
        out = np.zeros((self.H, self.d), np.float32)
        rc = lib().absp_oracle_attend(np.ascontiguousarray(q, np.float32), self.k_pool, self.v_pool,
                                      self.pool_pages, self.page_table, self.n, self.H, self.d, self.P,
                                      self.block_sizes, blocks, max_k, counts, out)
        if rc:
            raise ValueError("sparse_attention: invalid selection")
        return out

    def full_attention(self, q: np.ndarray) -> np.ndarray:
        out = np.zeros((self.H, self.d), np.float32)
        lib().absp_oracle_full_attention(np.ascontiguousarray(q, np.float32), self.k_pool, self.v_pool,
                                         self.pool_pages, self.page_table, self.n, self.H, self.d, self.P, out)
        return out

    def keys_logical(self) -> np.ndarray:
        """fp32 keys [H][n][d] in token order (what the reference's cache holds)."""
        return self._logical(self.k_pool)

    def values_logical(self) -> np.ndarray:
        return self._logical(self.v_pool)

    def _logical(self, pool):
        t = np.arange(self.n)
        pages = self.page_table[t // self.P]
        rows = pool[:, pages, t % self.P, :]  # [H][n][d]
        return np.ascontiguousarray(bf16_to_f32(rows))


def group_sum(qg: np.ndarray, H: int, G: int) -> np.ndarray:
    """fp32 left-to-right sum over each GQA group.
    qg: fp32 [H*G][d] -> [H][d]."""
    qg = np.asarray(qg, np.float32).reshape(H, G, -1)
    acc = qg[:, 0, :].copy()
    for g in range(1, G):
        acc = (acc + qg[:, g, :]).astype(np.float32)
    return acc


def oracle_decode(seq: OracleSeq, q_heads: np.ndarray, G: int, token_budget: int):
    """One GQA decode step of one sequence with the C restatement.
    q_heads: fp32 [H*G][d]. Returns (scores, selection, out[H*G][d])."""
    H, d = seq.H, seq.d
    qs = group_sum(q_heads, H, G)
    sc = seq.scores(qs)
    sel = seq.select(sc, token_budget)
    out = np.zeros((H * G, d), np.float32)
    qg = np.asarray(q_heads, np.float32).reshape(H, G, d)
    for g in range(G):
        out.reshape(H, G, d)[:, g, :] = seq.attend(np.ascontiguousarray(qg[:, g, :]), sel)
    return sc, sel, out


# ---------------------------------------------------------------------------
# The unmodified reference (oracle/_ref) on the same data
# ---------------------------------------------------------------------------
class RefSeq:
    """One sequence built by the reference itself: PagedKVCache::append per token,
    compute_block_centroids, quantize_store (ref_shim.cpp)."""

    def __init__(self, keys, values, P, block_sizes, method=0, bits=4, mode=1, capacity=0):
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
        self.H, self.n, self.d = keys.shape
        self.P = P
        bs = (_sz * self.H)(*[int(b) for b in block_sizes])
        h = C.c_void_p()
        _rcheck(ref().ref_seq_create(self.H, self.d, P, self.n, max(capacity, self.n), keys, values, bs,
                                     method, bits, mode, C.byref(h)))
        self.h = h
        self.method, self.bits = method, bits
        self.offsets = np.zeros(self.H + 1, np.uint64)
        ref().ref_seq_offsets(self.h, self.offsets)

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_seq_destroy(self.h)
            self.h = None

    @property
    def total(self) -> int:
        return int(self.offsets[-1])

    def store(self):
        t, d = self.total, self.d
        mm = self.method == 1
        out = {"values": np.zeros((t, d), np.float32)}
        if mm:
            out["values_min"] = np.zeros((t, d), np.float32)
        if self.bits:
            out["codes"] = np.zeros((t, d), np.uint8)
            out["scales"] = np.zeros((self.H, d), np.float32)
            out["zps"] = np.zeros((self.H, d), np.float32)
            if mm:
                out["codes_min"] = np.zeros((t, d), np.uint8)
                out["scales_min"] = np.zeros((self.H, d), np.float32)
                out["zps_min"] = np.zeros((self.H, d), np.float32)
        p = lambda k: out[k].ctypes.data if k in out else None
        _rcheck(ref().ref_seq_store(self.h, p("values"), p("values_min"), p("codes"), p("codes_min"),
                                    p("scales"), p("zps"), p("scales_min"), p("zps_min")))
        return out

    def scores(self, q) -> np.ndarray:
        out = np.zeros(self.total, np.float32)
        _rcheck(ref().ref_seq_estimate(self.h, np.ascontiguousarray(q, np.float32), out))
        return out

    def select(self, scores, token_budget):
        max_k = max(self.total, 1)
        blocks = np.zeros((self.H, max_k), np.uint32)
        counts = np.zeros(self.H, np.uint32)
        budgets = np.zeros(self.H, np.uint32)
        _rcheck(ref().ref_seq_select(self.h, np.ascontiguousarray(scores, np.float32), token_budget,
                                     blocks, max_k, counts, budgets))
        return [blocks[h, : counts[h]].copy() for h in range(self.H)]

    def attend(self, q) -> np.ndarray:
        """sparse_attention over the selection of the last select() call."""
        out = np.zeros((self.H, self.d), np.float32)
        _rcheck(ref().ref_seq_attend(self.h, np.ascontiguousarray(q, np.float32), out))
        return out

    def full_attention(self, q) -> np.ndarray:
        out = np.zeros((self.H, self.d), np.float32)
        _rcheck(ref().ref_seq_full_attention(self.h, np.ascontiguousarray(q, np.float32), out))
        return out

    def full_attention_weights(self, q):
        """full_attention_oracle: (output [H][d] fp32, weights [H][n] fp64)."""
        out = np.zeros((self.H, self.d), np.float32)
        w = np.zeros((self.H, self.n), np.float64)
        _rcheck(ref().ref_seq_full_attention_w(self.h, np.ascontiguousarray(q, np.float32), out, w))
        return out, w

    def decode_gqa(self, q_heads, G, token_budget) -> np.ndarray:
        out = np.zeros((self.H * G, self.d), np.float32)
        _rcheck(ref().ref_seq_decode_gqa(self.h, np.ascontiguousarray(q_heads, np.float32), G,
                                         token_budget, out))
        return out


class RefEngine:
    """The reference's own DecodeEngine (engine.hpp:99-129, via ref_shim.cpp): prefill,
    step (append + refresh_tail_centroids + requantize_heads + estimate -> select ->
    attend, or the fp64 full attention while seq_len <= T) and a store snapshot."""

    def __init__(self, H, d, P, candidates, token_budget, block_sizes, capacity, method=0, bits=4, mode=1):
        self.H, self.d = H, d
        self.max_k = int(token_budget // min(candidates) + 1)
        cands = (_sz * len(candidates))(*[int(c) for c in candidates])
        bs = (_sz * H)(*[int(b) for b in block_sizes])
        h = C.c_void_p()
        _rcheck(ref().ref_engine_create(H, d, P, cands, len(candidates), token_budget, method, bits, mode, bs,
                                        capacity, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_engine_destroy(self.h)
            self.h = None

    def prefill(self, keys, values, num_tokens):
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
        _rcheck(ref().ref_engine_prefill(self.h, keys, values, num_tokens, keys.shape[1]))

    def step(self, k, v, q):
        out = np.zeros((self.H, self.d), np.float32)
        blocks = np.zeros((self.H, self.max_k), np.uint32)
        counts = np.zeros(self.H, np.uint32)
        fb = C.c_int()
        _rcheck(ref().ref_engine_step(self.h, np.ascontiguousarray(k, np.float32), np.ascontiguousarray(v, np.float32),
                                      np.ascontiguousarray(q, np.float32), out, blocks.ctypes.data, self.max_k,
                                      counts.ctypes.data, C.byref(fb)))
        return out, [blocks[h, :counts[h]].copy() for h in range(self.H)], bool(fb.value)

    def store(self):
        total = _sz()
        _rcheck(ref().ref_engine_store(self.h, None, None, None, None, None, C.byref(total)))
        t = int(total.value)
        offsets = np.zeros(self.H + 1, np.uint64)
        values = np.zeros((t, self.d), np.float32)
        codes = np.zeros((t, self.d), np.uint8)
        scales = np.zeros((self.H, self.d), np.float32)
        zps = np.zeros((self.H, self.d), np.float32)
        _rcheck(ref().ref_engine_store(self.h, offsets.ctypes.data, values.ctypes.data, codes.ctypes.data,
                                       scales.ctypes.data, zps.ctypes.data, None))
        return dict(offsets=offsets, values=values, codes=codes, scales=scales, zps=zps)


def ref_generate_synthetic(n, H, d, profiles, signal=8.0, seed=0, scatter_gap=64):
    """generate_synthetic (workload.cpp:192-249). profiles: list of ("uniform",) |
    ("clustered", count, width) | ("scattered", hot). Returns keys, values [H][n][d], queries [H][d]."""
    kinds = (C.c_int * H)()
    a = (_sz * H)()
    b = (_sz * H)()
    for h, p in enumerate(profiles):
        if p[0] == "clustered":
            kinds[h], a[h], b[h] = 1, p[1], p[2]
        elif p[0] == "scattered":
            kinds[h], a[h] = 2, p[1]
    keys = np.zeros((H, n, d), np.float32)
    vals = np.zeros((H, n, d), np.float32)
    qs = np.zeros((H, d), np.float32)
    _rcheck(ref().ref_generate_synthetic(n, H, d, kinds, a, b, signal, seed, scatter_gap, keys, vals, qs))
    return keys, vals, qs


# ---------------------------------------------------------------------------
# Trace I/O and calibration of the unmodified reference (workload.cpp, calibrator.cpp)
# ---------------------------------------------------------------------------
def ref_save_trace(path, keys, values, queries, seed=0):
    keys = np.ascontiguousarray(keys, np.float32)
    H, n, d = keys.shape
    _rcheck(ref().ref_save_trace(str(path).encode(), H, d, n, seed, keys,
                                 np.ascontiguousarray(values, np.float32), np.ascontiguousarray(queries, np.float32)))


def ref_load_trace(path):
    """(keys [H][n][d], values, queries [H][d], seed) read by the reference's load_trace."""
    dims = np.zeros(4, np.uint64)
    _rcheck(ref().ref_load_trace(str(path).encode(), dims, None, None, None))
    H, d, n, seed = (int(x) for x in dims)
    k = np.zeros((H, n, d), np.float32)
    v = np.zeros((H, n, d), np.float32)
    q = np.zeros((H, d), np.float32)
    _rcheck(ref().ref_load_trace(str(path).encode(), dims, k.ctypes.data, v.ctypes.data, q.ctypes.data))
    return k, v, q, seed


def _calib_args(H, d, P, cands, T, method, bits, mode):
    return (H, d, P, (_sz * len(cands))(*cands), len(cands), T, method, bits, mode)


def ref_profile_sensitivity(keys, values, queries, P, cands, T, method=0, bits=4, mode=1):
    """keys/values [S][H][n][d], queries [S][H][d] -> recalls [H][len(cands)]."""
    keys = np.ascontiguousarray(keys, np.float32)
    S, H, n, d = keys.shape
    out = np.zeros((H, len(cands)), np.float64)
    _rcheck(ref().ref_profile_sensitivity(*_calib_args(H, d, P, cands, T, method, bits, mode), S, n, keys,
                                          np.ascontiguousarray(values, np.float32),
                                          np.ascontiguousarray(queries, np.float32), out))
    return out


def ref_transfer_check(block_sizes, keys, values, queries, P, cands, T, method=0, bits=4, mode=1):
    """-> dict(adaptive_recall, delta, avg_block_size, matched_candidate, uniform_recalls)."""
    keys = np.ascontiguousarray(keys, np.float32)
    S, H, n, d = keys.shape
    out = np.zeros(4 + len(cands), np.float64)
    _rcheck(ref().ref_transfer_check(*_calib_args(H, d, P, cands, T, method, bits, mode),
                                     (_sz * H)(*block_sizes), S, n, keys, np.ascontiguousarray(values, np.float32),
                                     np.ascontiguousarray(queries, np.float32), out))
    return dict(adaptive_recall=out[0], delta=out[1], avg_block_size=out[2], matched_candidate=int(out[3]),
                uniform_recalls=list(out[4:]))


def ref_assign_block_sizes(recalls, cands, tau):
    recalls = np.ascontiguousarray(recalls, np.float64)
    H = recalls.shape[0]
    out = (_sz * H)()
    _rcheck(ref().ref_assign_block_sizes(H, (_sz * len(cands))(*cands), len(cands), recalls, tau, out))
    return [int(x) for x in out]


def ref_write_recall_csv(path, recalls, cands, tag):
    recalls = np.ascontiguousarray(recalls, np.float64)
    _rcheck(ref().ref_write_recall_csv(str(path).encode(), recalls.shape[0], (_sz * len(cands))(*cands), len(cands),
                                       recalls, tag.encode()))


def ref_write_min_block_csv(path, sizes, tag):
    _rcheck(ref().ref_write_min_block_csv(str(path).encode(), (_sz * len(sizes))(*sizes), len(sizes), tag.encode()))
