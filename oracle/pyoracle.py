"""TEST INFRASTRUCTURE ONLY — Python bindings of the CPU checkers.

* ``Ref``  : oracle/_ref/libmagref.so, the reference's own sources compiled
             unmodified (naive_search, Aho–Corasick, maps, encode_text,
             superimposition) — see oracle/ref_driver.cpp.
* ``Port`` : oracle/libmagoracle.so, the plain-C restatement of the pieces the
             reference ships without bodies (filter machine, verifier, engine,
             tuner) — see oracle/mag_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
arm may import this module.  The product (paper_1405_5483_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmagref.so")
PORT_SO = os.path.join(HERE, "libmagoracle.so")

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
szp = C.POINTER(C.c_size_t)


def _pack(patterns: Sequence[bytes]):
    data = b"".join(patterns)
    buf = np.frombuffer(data if data else b"\0", dtype=np.uint8).copy()
    lens = np.array([len(p) for p in patterns] or [0], dtype=np.uintp)
    return buf, lens


def _u8(x) -> np.ndarray:
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x.view(np.uint8).reshape(-1))
    b = bytes(x)
    return np.frombuffer(b if b else b"\0", dtype=np.uint8)[: len(b)].copy() if b else np.zeros(0, np.uint8)


def _ptr(a: np.ndarray, t=u8p):
    if a.size == 0:
        a = np.zeros(1, dtype=a.dtype)
    return a.ctypes.data_as(t)


def ensure_port_built() -> str:
    if not os.path.exists(PORT_SO):
        subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
    return PORT_SO


class _Result:
    @staticmethod
    def take(lib, offs, pids, count):
        n = count.value
        o = np.ctypeslib.as_array(offs, shape=(max(n, 1),))[:n].copy() if n else np.zeros(0, np.uint64)
        p = np.ctypeslib.as_array(pids, shape=(max(n, 1),))[:n].copy() if n else np.zeros(0, np.uint32)
        lib_free = getattr(lib, "ref_free", None) or getattr(lib, "mo_free")
        lib_free(C.cast(offs, C.c_void_p))
        lib_free(C.cast(pids, C.c_void_p))
        return o.astype(np.uint64), p.astype(np.uint32)


class Ref:
    """The reference's compiled oracles (oracles.cpp:9-99) and host pieces."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (oracle/Makefile needs /root/reference)")
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_naive_search.argtypes = [u8p, C.c_size_t, u8p, szp, C.c_size_t,
                                       C.POINTER(u64p), C.POINTER(u32p), szp]
        L.ref_ac_search.argtypes = [u8p, C.c_size_t, u8p, szp, C.c_size_t, C.c_int,
                                    C.POINTER(u64p), C.POINTER(u32p), szp]
        L.ref_alphabet_map.argtypes = [C.c_int, u8p, szp, C.c_size_t, u8p, C.c_size_t, C.c_uint32,
                                       C.c_uint, u8p, u32p]
        L.ref_alphabet_map_hist.argtypes = [C.c_int, u64p, C.c_uint32, C.c_uint, u8p, u32p]
        L.ref_encode_text_strategy.argtypes = [C.c_int, u8p, szp, C.c_size_t, C.c_uint32, C.c_uint,
                                               C.c_uint, u8p, C.c_size_t, u32p]
        L.ref_classes.argtypes = [C.c_int, u8p, szp, C.c_size_t, C.c_uint32, C.c_uint, C.c_uint,
                                  C.c_int, szp, C.POINTER(u64p), C.POINTER(u32p)]
        L.ref_class_match_count.argtypes = [C.c_int, u8p, szp, C.c_size_t, C.c_uint32, C.c_uint,
                                            C.c_uint, u64p, C.POINTER(C.c_int)]
        L.ref_validate.argtypes = [u8p, szp, C.c_size_t, szp, szp, C.POINTER(C.c_long)]
        self.L = L

    def _err(self):
        return self.L.ref_last_error().decode()

    def naive(self, text, patterns):
        t = _u8(text)
        b, l = _pack(patterns)
        offs, pids, cnt = u64p(), u32p(), C.c_size_t()
        rc = self.L.ref_naive_search(_ptr(t), t.size, _ptr(b), _ptr(l, szp), len(patterns),
                                     C.byref(offs), C.byref(pids), C.byref(cnt))
        if rc:
            raise ValueError(self._err())
        return _Result.take(self.L, offs, pids, cnt)

    def ac(self, text, patterns, threads: int = 1):
        t = _u8(text)
        b, l = _pack(patterns)
        offs, pids, cnt = u64p(), u32p(), C.c_size_t()
        rc = self.L.ref_ac_search(_ptr(t), t.size, _ptr(b), _ptr(l, szp), len(patterns), threads,
                                  C.byref(offs), C.byref(pids), C.byref(cnt))
        if rc:
            raise ValueError(self._err())
        return _Result.take(self.L, offs, pids, cnt)

    def alphabet_map(self, strategy: int, patterns, sigma_prime: int, lowbits: int = 0, sample=None):
        b, l = _pack(patterns)
        s = _u8(sample) if sample is not None else np.zeros(0, np.uint8)
        table = (C.c_uint8 * 256)()
        sp = C.c_uint32()
        rc = self.L.ref_alphabet_map(strategy, _ptr(b), _ptr(l, szp), len(patterns), _ptr(s), s.size,
                                     sigma_prime, lowbits, table, C.byref(sp))
        if rc:
            raise ValueError(self._err())
        return bytes(table), sp.value

    def alphabet_map_hist(self, strategy: int, counts, sigma_prime: int, lowbits: int = 0):
        c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
        table = (C.c_uint8 * 256)()
        sp = C.c_uint32()
        rc = self.L.ref_alphabet_map_hist(strategy, _ptr(c, u64p), sigma_prime, lowbits, table, C.byref(sp))
        if rc:
            raise ValueError(self._err())
        return bytes(table), sp.value

    def encode_text(self, strategy, patterns, sigma_prime, lowbits, q, text):
        b, l = _pack(patterns)
        t = _u8(text)
        out = np.zeros(max(t.size // q, 1), dtype=np.uint32)
        rc = self.L.ref_encode_text_strategy(strategy, _ptr(b), _ptr(l, szp), len(patterns), sigma_prime,
                                             lowbits, q, _ptr(t), t.size, _ptr(out, u32p))
        if rc:
            raise ValueError(self._err())
        return out[: t.size // q]

    def classes(self, strategy, patterns, sigma_prime, lowbits, q, overlapping=False):
        b, l = _pack(patterns)
        length, csr, codes = C.c_size_t(), u64p(), u32p()
        rc = self.L.ref_classes(strategy, _ptr(b), _ptr(l, szp), len(patterns), sigma_prime, lowbits, q,
                                1 if overlapping else 0, C.byref(length), C.byref(csr), C.byref(codes))
        if rc:
            raise ValueError(self._err())
        n = length.value
        c = np.ctypeslib.as_array(csr, shape=(n + 1,)).copy()
        flat = np.ctypeslib.as_array(codes, shape=(max(int(c[-1]), 1),)).copy()
        self.L.ref_free(C.cast(csr, C.c_void_p))
        self.L.ref_free(C.cast(codes, C.c_void_p))
        return [flat[c[i]:c[i + 1]].tolist() for i in range(n)]

    def class_match_count(self, strategy, patterns, sigma_prime, lowbits, q):
        b, l = _pack(patterns)
        v, sat = C.c_uint64(), C.c_int()
        rc = self.L.ref_class_match_count(strategy, _ptr(b), _ptr(l, szp), len(patterns), sigma_prime,
                                          lowbits, q, C.byref(v), C.byref(sat))
        if rc:
            raise ValueError(self._err())
        return v.value, bool(sat.value)

    def validate(self, patterns):
        b, l = _pack(patterns)
        mn, mx, bad = C.c_size_t(), C.c_size_t(), C.c_long()
        rc = self.L.ref_validate(_ptr(b), _ptr(l, szp), len(patterns), C.byref(mn), C.byref(mx), C.byref(bad))
        if rc == 0:
            return ("ok", mn.value, mx.value)
        if rc == 1:
            return ("validation_error", bad.value, self._err())
        raise ValueError(self._err())


class _MoParams(C.Structure):
    _fields_ = [
        ("variant", C.c_int), ("gram_mode", C.c_int), ("q", C.c_uint), ("k", C.c_uint),
        ("word_bits", C.c_uint), ("table_bits", C.c_uint), ("sigma_prime", C.c_uint32),
        ("window_rule", C.c_int), ("probes", C.c_uint), ("blocks", C.c_uint), ("map", C.c_uint8 * 256),
    ]


class _MoShape(C.Structure):
    _fields_ = [("entries", C.c_uint64), ("L", C.c_size_t), ("k", C.c_uint), ("m_prime", C.c_uint),
                ("match_mask", C.c_uint64), ("boundary_keep", C.c_uint64)]


class _MoTuneIn(C.Structure):
    _fields_ = [("sigma", C.c_uint32), ("sigma_prime", C.c_uint32), ("r", C.c_uint64), ("m", C.c_uint64),
                ("n", C.c_uint64), ("word_bits", C.c_uint32)]


class _MoTuneOut(C.Structure):
    _fields_ = [("q", C.c_int), ("k", C.c_int), ("sigma_prime", C.c_int), ("rho", C.c_double),
                ("predicted_p", C.c_double), ("predicted_cost", C.c_double)]


class Port:
    """The C restatement of the reference search phase (oracle/mag_oracle.c)."""

    def __init__(self, path: Optional[str] = None):
        path = path or ensure_port_built()
        L = C.CDLL(path)
        L.mo_free.argtypes = [C.c_void_p]
        L.mo_search.argtypes = [u8p, C.c_size_t, u8p, szp, C.c_size_t, C.POINTER(_MoParams),
                                C.POINTER(u64p), C.POINTER(u32p), szp, u64p, u64p]
        L.mo_naive_search.argtypes = [u8p, C.c_size_t, u8p, szp, C.c_size_t, C.POINTER(u64p),
                                      C.POINTER(u32p), szp]
        L.mo_map_build.argtypes = [C.c_int, u64p, C.c_uint32, C.c_uint, u8p, u32p]
        L.mo_encode_text.argtypes = [u8p, C.c_uint32, C.c_uint, u8p, C.c_size_t, u32p]
        L.mo_gram_hash.argtypes = [u8p, C.c_uint]
        L.mo_gram_hash.restype = C.c_uint32
        L.mo_machine_shape.argtypes = [C.POINTER(_MoParams), C.c_size_t, C.POINTER(_MoShape)]
        L.mo_build_masks.argtypes = [C.POINTER(_MoParams), u8p, szp, C.c_size_t, C.POINTER(_MoShape), u64p]
        for f in ("mo_expected_class_size", "mo_match_probability"):
            getattr(L, f).argtypes = [C.c_double, C.c_double]
            getattr(L, f).restype = C.c_double
        L.mo_tune.argtypes = [C.POINTER(_MoTuneIn), C.c_int, C.c_int, C.POINTER(_MoTuneOut)]
        L.mo_choose_q.argtypes = [C.POINTER(_MoTuneIn)]
        L.mo_choose_q.restype = C.c_uint
        L.mo_choose_k.argtypes = [C.POINTER(_MoTuneIn), C.c_uint]
        L.mo_choose_k.restype = C.c_uint
        L.mo_strided_k_seed.argtypes = [C.POINTER(_MoTuneIn), C.c_uint]
        L.mo_strided_k_seed.restype = C.c_double
        L.mo_predicted_cost.argtypes = [C.POINTER(_MoTuneIn), C.c_uint, C.c_uint]
        L.mo_predicted_cost.restype = C.c_double
        L.mo_resolve_sigma_prime.argtypes = [C.c_uint32, C.c_uint32]
        L.mo_resolve_sigma_prime.restype = C.c_uint32
        L.mo_sample_offsets.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, u64p]
        self.L = L

    @staticmethod
    def params(variant=0, gram_mode=0, q=1, k=1, word_bits=64, table_bits=0, sigma_prime=256,
               table: Optional[bytes] = None, window_rule=0, probes=1, blocks=0) -> _MoParams:
        p = _MoParams()
        p.probes = probes
        p.blocks = blocks
        p.variant, p.gram_mode, p.q, p.k = variant, gram_mode, q, k
        p.word_bits, p.table_bits, p.sigma_prime, p.window_rule = word_bits, table_bits, sigma_prime, window_rule
        t = table if table is not None else bytes(range(256))
        for i in range(256):
            p.map[i] = t[i]
        return p

    def search(self, text, patterns, P: _MoParams):
        t = _u8(text)
        b, l = _pack(patterns)
        offs, pids, cnt = u64p(), u32p(), C.c_size_t()
        reads, cands = C.c_uint64(), C.c_uint64()
        rc = self.L.mo_search(_ptr(t), t.size, _ptr(b), _ptr(l, szp), len(patterns), C.byref(P), C.byref(offs),
                              C.byref(pids), C.byref(cnt), C.byref(reads), C.byref(cands))
        if rc:
            raise ValueError(f"mo_search failed: {rc}")
        o, p = _Result.take(self.L, offs, pids, cnt)
        return o, p, reads.value, cands.value

    def naive(self, text, patterns):
        t = _u8(text)
        b, l = _pack(patterns)
        offs, pids, cnt = u64p(), u32p(), C.c_size_t()
        self.L.mo_naive_search(_ptr(t), t.size, _ptr(b), _ptr(l, szp), len(patterns), C.byref(offs),
                               C.byref(pids), C.byref(cnt))
        return _Result.take(self.L, offs, pids, cnt)

    def map_build(self, strategy, counts, sigma_prime, lowbits=0):
        c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
        table = (C.c_uint8 * 256)()
        sp = C.c_uint32()
        rc = self.L.mo_map_build(strategy, _ptr(c, u64p), sigma_prime, lowbits, table, C.byref(sp))
        if rc:
            raise ValueError("config error")
        return bytes(table), sp.value

    def encode_text(self, table: bytes, sigma_prime, q, text):
        t = _u8(text)
        tb = np.frombuffer(table, dtype=np.uint8).copy()
        out = np.zeros(max(t.size // q, 1), dtype=np.uint32)
        self.L.mo_encode_text(_ptr(tb), sigma_prime, q, _ptr(t), t.size, _ptr(out, u32p))
        return out[: t.size // q]

    def gram_hash(self, gram: bytes) -> int:
        g = _u8(gram)
        return int(self.L.mo_gram_hash(_ptr(g), len(gram)))

    def masks(self, patterns, P: _MoParams):
        b, l = _pack(patterns)
        m = min(len(p) for p in patterns)
        S = _MoShape()
        rc = self.L.mo_machine_shape(C.byref(P), m, C.byref(S))
        if rc:
            raise ValueError("config error")
        out = np.zeros(S.entries, dtype=np.uint64)
        self.L.mo_build_masks(C.byref(P), _ptr(b), _ptr(l, szp), len(patterns), C.byref(S), _ptr(out, u64p))
        return out, {"entries": S.entries, "L": S.L, "k": S.k, "m_prime": S.m_prime,
                     "match_mask": S.match_mask}

    def tune(self, sigma, r, m, n=1 << 20, sigma_prime=0, word_bits=0, fixed_q=0, fixed_k=0):
        ti = _MoTuneIn(sigma, sigma_prime, r, m, n, word_bits)
        to = _MoTuneOut()
        rc = self.L.mo_tune(C.byref(ti), fixed_q, fixed_k, C.byref(to))
        if rc:
            raise ValueError("config error")
        return {f: getattr(to, f) for f, _ in _MoTuneOut._fields_}

    def sample_offsets(self, corpus_len, count, length, seed):
        out = np.zeros(max(count, 1), dtype=np.uint64)
        rc = self.L.mo_sample_offsets(corpus_len, count, length, seed, _ptr(out, u64p))
        if rc:
            raise ValueError("config error")
        return out[:count]


def as_pairs(offs, pids):
    return list(zip([int(x) for x in offs], [int(x) for x in pids]))


# ---------------------------------------------------------------- roll --
# Restatement of the GPU's dense rolling-hash filter (a GPU extension, not a
# reference algorithm: paper_1405_5483_b200/csrc/mag_common.h roll_*), used
# to check the roll kernel's Bloom table and its candidate counter.
ROLL_B = 0x9E3779B1


def roll_hashes(text, q: int) -> np.ndarray:
    """H(p) = sum_{j<q} t[p+j] * B^(q-1-j) mod 2^32 for every p <= n - q."""
    t = _u8(text).astype(np.uint32)
    n = t.size - q + 1
    if n <= 0:
        return np.zeros(0, dtype=np.uint32)
    h = np.zeros(n, dtype=np.uint32)
    with np.errstate(over="ignore"):
        for j in range(q):
            h = h * np.uint32(ROLL_B) + t[j:j + n]
    return h


ROLL_PROBE_MUL = {1: 0x85EBCA77, 2: 0xC2B2AE3D}


def _roll_slots(h: np.ndarray, words: int, probes: int):
    g = h.astype(np.uint32)  # the hash itself picks the word (top bits) and probe 0 (low bits)
    w = ((g.astype(np.uint64) * np.uint64(words)) >> np.uint64(32)).astype(np.int64)
    shifts = [g] + [((h.astype(np.uint64) * np.uint64(ROLL_PROBE_MUL[i])) >> np.uint64(32)).astype(np.uint32)
                    for i in range(1, probes)]
    bits = [(np.uint32(31) - (s & np.uint32(31))).astype(np.uint32) for s in shifts]
    return w, bits


def roll_bloom(patterns, q: int, words: int, probes: int) -> np.ndarray:
    """The Bloom words the host builds (bit set = present)."""
    keys = np.array([roll_hashes(p[:q], q)[0] for p in patterns], dtype=np.uint32)
    w, bits = _roll_slots(keys, words, probes)
    out = np.zeros(words, dtype=np.uint32)
    for b in bits:
        np.bitwise_or.at(out, w, np.uint32(1) << b)
    return out


def roll_candidates(text, patterns, q: int, words: int, probes: int) -> int:
    """Positions p <= n - q whose rolling hash passes the Bloom filter."""
    table = roll_bloom(patterns, q, words, probes)
    h = roll_hashes(text, q)
    w, bits = _roll_slots(h, words, probes)
    ok = np.ones(h.size, dtype=bool)
    for b in bits:
        ok &= ((table[w] >> b) & np.uint32(1)).astype(bool)
    return int(ok.sum())


# ---------------------------------------------------------------- pack2 --
# Restatement of the GPU's two-level 2-bit-code filter (a GPU plan of the
# reference's sigma' = 4 exact q-gram codes, qgram.hpp:30-36; see
# paper_1405_5483_b200/csrc/scan_pack2.cu): level 1 is the set of the
# patterns' first-10-symbol codes; a position p <= n - q is a candidate when
# its own first-10-symbol code is in that set.
def pack2_codes(text, length: int, shift: int) -> np.ndarray:
    """code(p) = sum_{i<length} ((t[p+i] >> shift) & 3) << 2i for p <= n - length."""
    t = _u8(text).astype(np.uint32)
    n = t.size - length + 1
    if n <= 0:
        return np.zeros(0, dtype=np.uint32)
    s = (t >> np.uint32(shift)) & np.uint32(3)
    c = np.zeros(n, dtype=np.uint32)
    for i in range(length):
        c |= s[i:i + n] << np.uint32(2 * i)
    return c


def pack2_candidates(text, patterns, q: int, shift: int) -> int:
    keys = np.unique(np.array([pack2_codes(p[:10], 10, shift)[0] for p in patterns], dtype=np.uint32))
    t = _u8(text)
    n = t.size - q + 1
    if n <= 0:
        return 0
    codes = pack2_codes(t[: n + 9], 10, shift)[:n]
    return int(np.isin(codes, keys).sum())
