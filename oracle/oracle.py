"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes front end over the two CPU checkers of the hipprune hot path:

* ``Oracle("port")``      -> oracle/liboracle.so, the plain-C restatement
  (oracle/hipprune_oracle.c) of the reference algorithm;
* ``Oracle("reference")`` -> oracle/_ref/libhipref.so, the unmodified reference
  library compiled from /root/reference/proj/src plus oracle/ref_shim.cpp.

Both expose the same functions with the same argument meaning. Only tests/,
``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference``
legs may import this module, and only as the checker or the CPU baseline.

Array conventions: q ``[n_heads, rows, d]`` fp32, k/v ``[n_kv, t_kv, d]`` fp32,
q-head h reads kv-head ``h // (n_heads // n_kv)``; index lists are int64.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libhipref.so"
REF_SRC = Path("/root/reference/proj")

_sz = C.c_size_t
_i64p = C.POINTER(C.c_int64)
_f32p = C.POINTER(C.c_float)
_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)
_vp = C.c_void_p

_ERRORS = {1: "ContractViolation", 2: "ValueError", 3: "IndexError", 4: "LogicError",
           5: "RuntimeError", 6: "PartialCommitError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{_ERRORS.get(code, code)}] {msg}")
        self.code = code
        self.kind = _ERRORS.get(code, str(code))


def build(kind: str = "all") -> None:
    """Compile the checkers (make -C oracle). The reference leg needs /root/reference."""
    targets = ["oracle"]
    if kind in ("all", "ref") and REF_SRC.exists():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def available(kind: str) -> bool:
    return (PORT_SO if kind == "port" else REF_SO).exists()


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a, t):
    return a.ctypes.data_as(t)


def _szarr(vals):
    arr = (C.c_size_t * max(1, len(vals)))(*vals)
    return arr


class Oracle:
    _cache: dict = {}

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not path.exists():
            if kind == "port" or REF_SRC.exists():
                build("ref" if kind != "port" else "port")
        if not path.exists():
            raise FileNotFoundError(f"oracle library missing: {path}")
        key = str(path)
        if key not in Oracle._cache:
            Oracle._cache[key] = C.CDLL(key)
        self.lib = Oracle._cache[key]
        self.pre = "orc_" if kind == "port" else "ref_"
        self._setup()

    def _fn(self, name, restype, *argtypes):
        f = getattr(self.lib, self.pre + name)
        f.restype = restype
        f.argtypes = list(argtypes)
        return f

    def _setup(self):
        f = self._fn
        self.f_err = f("last_error", C.c_char_p)
        self.f_code = f("last_error_code", C.c_int)
        self.f_lcount = f("lists_count", _sz, _vp)
        self.f_llen = f("lists_len", _sz, _vp, _sz)
        self.f_lget = f("lists_get", None, _vp, _sz, _i64p)
        self.f_lfree = f("lists_free", None, _vp)
        self.f_lfrom = f("lists_from", _vp, _i64p, _szp, _sz)
        self.f_rope = f("build_rope_table", C.c_int, _sz, _sz, C.c_float, _f32p, _f32p)
        self.f_stage = f("run_pruning_stage", _vp, _sz, _sz, _sz, _i64p, _sz, _f32p, _sz, _sz,
                         _f32p, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int, _sz, _sz, _u64p, _u64p)
        self.f_rep = f("select_rep", C.c_int, _f32p, _sz, _i64p, _sz, _f32p, _sz, _sz, _sz, _sz,
                       _sz, C.c_int, _sz, _sz, _sz, _sz, _i64p, _i64p, _szp)
        self.f_mask = f("build_mask", _vp, _f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _sz, _szp, _sz,
                        _sz, _sz, C.c_int, _sz, _sz, C.POINTER(_vp), _szp, _szp)
        self.f_sel = f("selected_indices", _vp, _vp, _sz, _sz, _sz, _sz, _sz)
        self.f_row = f("attention_row", C.c_int, _f32p, _i64p, _sz, _sz, C.c_int, _f32p, _f32p,
                       _sz, _sz, _sz, _f32p)
        self.f_bsa = f("block_sparse_attention", C.c_int, _f32p, _f32p, _f32p, _sz, _sz, _sz, _sz,
                       _sz, _vp, _sz, _sz, _sz, _sz, C.c_int, _f32p)
        self.f_dense = f("dense_attention", C.c_int, _f32p, _f32p, _f32p, _sz, _sz, _sz, _sz, _f32p)
        self.f_topk = f("exact_topk", _vp, _f32p, _f32p, _sz, _sz, _sz)
        self.f_recall = f("attention_recall", C.c_double, _i64p, _sz, _f32p, _f32p, _sz, _sz)
        self.f_dec = f("decode_layer_step", C.c_int, _f32p, _f32p, _f32p, _sz, _sz, _sz, _sz, _szp,
                       _sz, _sz, _sz, C.c_int, _sz, _sz, _sz, C.c_int, _i64p, _sz, _szp, _f32p,
                       C.POINTER(C.c_double))
        self.f_snew = f("store_new", _vp, _sz, _sz, _sz, _sz)
        self.f_sfree = f("store_free", None, _vp)
        self.f_spage = f("store_page_of", C.c_int, _vp, _sz, _sz, _u64p)
        self.f_sacc = f("store_access", C.c_int, _vp, C.c_int, _u64p, _sz, _u64p, _szp)
        self.f_scom = f("store_commit", C.c_int, _vp, C.c_int, _u64p, _sz, _u64p, _szp)
        self.f_srec = f("store_recency", _sz, _vp, C.c_int, _u64p, _sz)
        self.f_sstat = f("store_stats", None, _vp, C.c_int, _u64p)
        self.f_schk = f("store_check", C.c_int, _vp)
        if self.kind == "reference":
            self.f_gen = f("generate", C.c_int, _sz, _sz, _sz, _sz, _sz, C.c_double, C.c_uint64,
                           _szp, _f32p, _sz, _f32p, _f32p, _f32p)
            self.f_counts = f("decode_read_counts", C.c_int, _f32p, _f32p, _sz, _sz, _sz, _szp,
                              _sz, _sz, _sz, C.c_int, _sz, _sz, _u64p, _u64p)
            self.f_enew = f("engine_new", _vp, _f32p, _f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _sz,
                            _szp, _sz, _sz, _sz, _szp, C.c_int, _sz, _sz, _sz, _sz, C.c_double,
                            C.c_double, _sz)
            self.f_efree = f("engine_free", None, _vp)
            self.f_eprefill = f("engine_prefill", _vp, _vp, _f32p)
            self.f_estep = f("engine_step", C.c_int, _vp, _sz, _f32p, C.POINTER(C.c_int),
                             C.POINTER(C.c_double), C.POINTER(C.c_double), _u64p, _szp)
            self.f_ecache = f("engine_stage_cache", _vp, _vp, _sz, _sz)
            self.f_efrozen = f("engine_set_frozen", C.c_int, _vp, C.POINTER(C.c_int), _sz)
            self.f_chash = f("config_hash", C.c_int, C.POINTER(C.c_char_p), _sz, _u64p)
            self.f_erecency = f("engine_store_recency", _sz, _vp, C.c_int, _u64p, _sz)

    # ---------------------------------------------------------------- helpers
    def _raise(self):
        raise OracleError(self.f_code(), self.f_err().decode())

    def _check(self, rc):
        if rc != 0:
            self._raise()

    def _take_lists(self, h) -> list[np.ndarray]:
        if not h:
            self._raise()
        try:
            out = []
            for i in range(self.f_lcount(h)):
                arr = np.empty(self.f_llen(h, i), dtype=np.int64)
                if arr.size:
                    self.f_lget(h, i, _p(arr, _i64p))
                out.append(arr)
            return out
        finally:
            self.f_lfree(h)

    def _make_lists(self, lists):
        lens = [len(l) for l in lists]
        flat = _i64(np.concatenate([np.asarray(l, dtype=np.int64) for l in lists]) if lists and sum(lens) else np.zeros(1, np.int64))
        lens_arr = _szarr(lens)
        h = self.f_lfrom(_p(flat, _i64p), lens_arr, len(lists))
        return h

    # ------------------------------------------------------------------- api
    def rope_table(self, max_pos: int, d: int, theta: float = 10000.0):
        cos = np.empty((max_pos, d // 2), np.float32)
        sin = np.empty((max_pos, d // 2), np.float32)
        self._check(self.f_rope(max_pos, d, theta, _p(cos, _f32p), _p(sin, _f32p)))
        return cos, sin

    def run_pruning_stage(self, stage, indices, q, k, *, layer1=4, stream=0, qstart=0,
                          ext=False, cutoff=3, rope_max=0, count_reads=False):
        """stage=(bq, lc, keep); q [H, rows, d]; k [H_kv, T, d]."""
        q = _f32(q); k = _f32(k); idx = _i64(indices)
        if idx.size == 0:
            idx = np.zeros(1, np.int64)
            n = 0
        else:
            n = idx.size
        H, rows, d = q.shape
        nkv, t, _ = k.shape
        tot, dis = C.c_uint64(0), C.c_uint64(0)
        h = self.f_stage(stage[0], stage[1], stage[2], _p(idx, _i64p), n, _p(q, _f32p), H, rows,
                         _p(k, _f32p), nkv, t, d, layer1, stream, qstart, int(ext), cutoff,
                         rope_max, C.byref(tot) if count_reads else None,
                         C.byref(dis) if count_reads else None)
        out = self._take_lists(h)[0]
        if count_reads:
            return out, int(tot.value), int(dis.value)
        return out

    def select_rep(self, q, chunk, k, *, layer1=4, stream=0, qstart=0, ext=False, cutoff=3,
                   chunk_index=0, chunk_count=1, rope_max=0):
        n = len(chunk)
        q = _f32(q); k = _f32(k); chunk = _i64(chunk) if n else np.zeros(1, np.int64)
        rows, d = q.shape
        t = k.shape[0]
        rep = C.c_int64(0)
        reads = np.zeros(4 * 64 + 8, np.int64)
        nr = C.c_size_t(0)
        self._check(self.f_rep(_p(q, _f32p), rows, _p(chunk, _i64p), n, _p(k, _f32p), t, d,
                               layer1, stream, qstart, int(ext), cutoff, chunk_index, chunk_count,
                               rope_max, C.byref(rep), _p(reads, _i64p), C.byref(nr)))
        return int(rep.value), reads[: nr.value].copy()

    def build_mask(self, q, k, stages, *, sink, stream, layer0=0, ext=False, cutoff=3, threads=1):
        """q [H, Tq, d], k [H_kv, Tkv, d]; returns (lists, trace, block_size, query_offset)."""
        q = _f32(q); k = _f32(k)
        H, tq, d = q.shape
        nkv, tkv, _ = k.shape
        st = _szarr([x for s in stages for x in s])
        tr = _vp()
        bs, off = C.c_size_t(0), C.c_size_t(0)
        h = self.f_mask(_p(q, _f32p), _p(k, _f32p), H, nkv, tq, tkv, d, layer0, st, len(stages),
                        sink, stream, int(ext), cutoff, threads, C.byref(tr), C.byref(bs),
                        C.byref(off))
        lists = self._take_lists(h)
        trace = self._take_lists(tr.value)
        return lists, trace, int(bs.value), int(off.value)

    def selected_indices(self, lists, block_size, sink, stream, offset, row):
        h = self._make_lists(lists)
        try:
            return self._take_lists(self.f_sel(h, block_size, sink, stream, offset, row))[0]
        finally:
            self.f_lfree(h)

    def attention_row(self, q_row, selected, pos, k, v, *, ext=False, rope_max=0):
        q = _f32(q_row); sel = _i64(selected); k = _f32(k); v = _f32(v)
        t, d = k.shape
        out = np.zeros(d, np.float32)
        self._check(self.f_row(_p(q, _f32p), _p(sel, _i64p), sel.size, pos, int(ext),
                               _p(k, _f32p), _p(v, _f32p), t, d, rope_max, _p(out, _f32p)))
        return out

    def block_sparse_attention(self, q, k, v, lists, *, block_size, sink, stream, offset, ext=False):
        q = _f32(q); k = _f32(k); v = _f32(v)
        H, tq, d = q.shape
        nkv, tkv, _ = k.shape
        out = np.zeros((H, tq, d), np.float32)
        h = self._make_lists(lists)
        try:
            self._check(self.f_bsa(_p(q, _f32p), _p(k, _f32p), _p(v, _f32p), H, nkv, tq, tkv, d, h,
                                   block_size, sink, stream, offset, int(ext), _p(out, _f32p)))
        finally:
            self.f_lfree(h)
        return out

    def dense_attention(self, q, k, v):
        q = _f32(q); k = _f32(k); v = _f32(v)
        H, tq, d = q.shape
        tkv = k.shape[1]
        out = np.zeros((H, tq, d), np.float32)
        self._check(self.f_dense(_p(q, _f32p), _p(k, _f32p), _p(v, _f32p), H, tq, tkv, d, _p(out, _f32p)))
        return out

    def exact_topk(self, q, keys, k):
        q = _f32(q); keys = _f32(keys)
        return self._take_lists(self.f_topk(_p(q, _f32p), _p(keys, _f32p), keys.shape[0], keys.shape[1], k))[0]

    def attention_recall(self, selected, q, keys):
        sel = _i64(selected) if len(selected) else np.zeros(1, np.int64)
        q = _f32(q); keys = _f32(keys)
        r = self.f_recall(_p(sel, _i64p), len(selected), _p(q, _f32p), _p(keys, _f32p), keys.shape[0], keys.shape[1])
        if r < 0:
            self._raise()
        return r

    def decode_layer_step(self, q, k, v, stages, *, sink, stream, ext=False, layer1=4, cutoff=3,
                          threads=1, kv_shared=False, cap=None):
        """q [G, hpm, d]; k, v [G, T, d] (or [T, d] with kv_shared). Returns
        (masks list per group, out [G, hpm, d], seconds)."""
        q = _f32(q); k = _f32(k); v = _f32(v)
        G, hpm, d = q.shape
        t = k.shape[-2]
        cap = cap or max(s[2] for s in stages)
        masks = np.zeros((G, cap), np.int64)
        lens = (C.c_size_t * G)()
        out = np.zeros((G, hpm, d), np.float32)
        secs = C.c_double(0)
        st = _szarr([x for s in stages for x in s])
        self._check(self.f_dec(_p(q, _f32p), _p(k, _f32p), _p(v, _f32p), G, hpm, t, d, st,
                               len(stages), sink, stream, int(ext), layer1, cutoff, threads,
                               int(kv_shared), _p(masks, _i64p), cap, lens, _p(out, _f32p),
                               C.byref(secs)))
        return [masks[g, : lens[g]].copy() for g in range(G)], out, secs.value

    # ----------------------------------------------------------- reference-only
    def generate(self, heads=1, layers=1, seq_kv=1024, seq_q=64, dim=32, locality=64.0, seed=1,
                 needles=()):
        assert self.kind == "reference", "generate needs the reference (libstdc++ <random>)"
        tq = seq_q or seq_kv
        q = np.empty((layers, heads, tq, dim), np.float32)
        k = np.empty((layers, heads, seq_kv, dim), np.float32)
        v = np.empty((layers, heads, seq_kv, dim), np.float32)
        pos = _szarr([p for p, _ in needles])
        strength = np.asarray([s for _, s in needles] or [0.0], np.float32)
        self._check(self.f_gen(heads, layers, seq_kv, seq_q, dim, locality, seed, pos,
                               _p(strength, _f32p), len(needles), _p(q, _f32p), _p(k, _f32p),
                               _p(v, _f32p)))
        return q, k, v

    def config_hash(self, overrides):
        """config.cpp config_hash over default_config() + overrides (report plumbing)."""
        arr = (C.c_char_p * max(1, len(overrides)))(*[o.encode() for o in overrides])
        out = np.zeros(1, np.uint64)
        self._check(self.f_chash(arr, len(overrides), _p(out, _u64p)))
        return int(out[0])

    def decode_read_counts(self, q, k, stages, *, sink, stream, ext=False, layer1=4, cutoff=3):
        """Distinct / total key-row reads per stage for one group (q [hpm, d], k [T, d])."""
        assert self.kind == "reference"
        q = _f32(q); k = _f32(k)
        hpm, d = q.shape
        t = k.shape[0]
        n = len(stages)
        dis = np.zeros(n, np.uint64); tot = np.zeros(n, np.uint64)
        st = _szarr([x for s in stages for x in s])
        self._check(self.f_counts(_p(q, _f32p), _p(k, _f32p), hpm, t, d, st, n, sink, stream,
                                  int(ext), layer1, cutoff, _p(dis, _u64p), _p(tot, _u64p)))
        return dis.astype(np.int64), tot.astype(np.int64)

    def engine(self, q, k, v, *, prefill_len, q_len, stages, sink, stream, refresh, ext=False,
               cutoff=3, page_size=16, mask_cap=64, sa_cap=64, dev_cost=1.0, host_cost=31.5):
        """The reference DecodeEngine (decode.cpp:104-289) over a full workload
        q, k, v [layers, heads, T, d] (one query per position)."""
        assert self.kind == "reference"
        return _Engine(self, q, k, v, prefill_len, q_len, stages, sink, stream, refresh, ext,
                       cutoff, page_size, mask_cap, sa_cap, dev_cost, host_cost)

    # ------------------------------------------------------------------ store
    def store(self, num_layers, page_size, mask_cap, sa_cap):
        return _Store(self, num_layers, page_size, mask_cap, sa_cap)


class _Engine:
    def __init__(self, o: Oracle, q, k, v, prefill_len, q_len, stages, sink, stream, refresh, ext,
                 cutoff, page_size, mask_cap, sa_cap, dev_cost=1.0, host_cost=31.5):
        self.o = o
        self.q, self.k, self.v = _f32(q), _f32(k), _f32(v)
        L, H, T, d = self.q.shape
        self.shape = (L, H, d)
        self.n_stages = len(stages)
        st = _szarr([x for s_ in stages for x in s_])
        rf = _szarr(list(refresh))
        self.h = o.f_enew(_p(self.q, _f32p), _p(self.k, _f32p), _p(self.v, _f32p), L, H, T, d,
                          prefill_len, q_len, st, len(stages), sink, stream, rf, int(ext), cutoff,
                          page_size, mask_cap, sa_cap, dev_cost, host_cost, 0)
        if not self.h:
            o._raise()

    def __del__(self):
        if getattr(self, "h", None):
            self.o.f_efree(self.h)
            self.h = None

    def prefill(self):
        h = self.o.f_eprefill(self.h, None)
        if not h:
            self.o._raise()
        return self.o._take_lists(h)

    def step(self, token_index):
        L, H, d = self.shape
        n = self.n_stages
        out = np.zeros((L, H, d), np.float32)
        refreshed = (C.c_int * n)()
        lat = (C.c_double * n)()
        bsa = C.c_double()
        c4 = np.zeros(4, np.uint64)
        sizes = (C.c_size_t * n)()
        self.o._check(self.o.f_estep(self.h, token_index, _p(out, _f32p), refreshed, lat,
                                     C.byref(bsa), _p(c4, _u64p), sizes))
        self.last_telemetry = {"stage_latency": list(lat), "bsa_latency": bsa.value,
                               "mask_hits": int(c4[0]), "mask_accesses": int(c4[1]),
                               "sa_hits": int(c4[2]), "sa_accesses": int(c4[3])}
        return out, [bool(x) for x in refreshed], list(sizes)

    def set_frozen_stages(self, frozen):
        arr = (C.c_int * len(frozen))(*[int(bool(x)) for x in frozen])
        self.o._check(self.o.f_efrozen(self.h, arr, len(frozen)))

    def store_recency(self, bank):
        n = self.o.f_erecency(self.h, bank, None, 0)
        out = np.zeros(max(1, n), np.uint64)
        self.o.f_erecency(self.h, bank, _p(out, _u64p), n)
        return [int(x) for x in out[:n]]

    def stage_cache(self, layer, stage):
        return self.o._take_lists(self.o.f_ecache(self.h, layer, stage))[0]


class _Store:
    MASK, SA = 0, 1

    def __init__(self, o: Oracle, num_layers, page_size, mask_cap, sa_cap):
        self.o = o
        self.h = o.f_snew(num_layers, page_size, mask_cap, sa_cap)
        if not self.h:
            o._raise()

    def __del__(self):
        if getattr(self, "h", None):
            self.o.f_sfree(self.h)
            self.h = None

    def page_of(self, layer, token):
        out = C.c_uint64(0)
        self.o._check(self.o.f_spage(self.h, layer, token, C.byref(out)))
        return int(out.value)

    def access(self, bank, pages):
        p = np.ascontiguousarray(pages, np.uint64)
        miss = np.zeros(max(1, p.size), np.uint64)
        n = C.c_size_t(0)
        self.o._check(self.o.f_sacc(self.h, bank, _p(p, _u64p), p.size, _p(miss, _u64p), C.byref(n)))
        return miss[: n.value].copy()

    def commit(self, bank, pages):
        p = np.ascontiguousarray(pages, np.uint64)
        ev = np.zeros(max(1, p.size), np.uint64)
        n = C.c_size_t(0)
        self.o._check(self.o.f_scom(self.h, bank, _p(p, _u64p), p.size, _p(ev, _u64p), C.byref(n)))
        return ev[: n.value].copy()

    def recency(self, bank):
        n = self.o.f_srec(self.h, bank, None, 0)
        out = np.zeros(max(1, n), np.uint64)
        self.o.f_srec(self.h, bank, _p(out, _u64p), n)
        return out[:n].copy()

    def stats(self, bank):
        out = np.zeros(3, np.uint64)
        self.o.f_sstat(self.h, bank, _p(out, _u64p))
        return tuple(int(x) for x in out)

    def check(self):
        self.o._check(self.o.f_schk(self.h))
