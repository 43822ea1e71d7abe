"""Python mirror of the mag C ABI served by libmag_b200.so (B200, sm_100a).

The reference exposes its search path only through ``proj/include/mag.h``
(engine create -> prepare text -> search -> sorted (offset, pattern_index)
matches).  This module binds exactly that ABI with ctypes and keeps its
names, argument meaning and error behaviour: every non-OK status raises
:class:`MagError` carrying the status and ``mag_last_error()``.

There is no CPU fallback: importing works anywhere, but a search needs the
in-tree ``libmag_b200.so`` and a CUDA device; otherwise it fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmag_b200.so")
# Profiling only (tools/): MAG_B200_PROFILE_LIB=diag loads the in-tree
# diagnostics build (`make diag`), whose searches honour MAG_B200_DIAG;
# MAG_B200_PROFILE_LIB=<name> loads libmag_b200_<name>.so (A/B builds).
if os.environ.get("MAG_B200_PROFILE_LIB"):
    LIB_PATH = os.path.join(_HERE, f"libmag_b200_{os.environ['MAG_B200_PROFILE_LIB']}.so")

# mag_status (mag.h:26-36)
MAG_OK = 0
MAG_ERR_NULL_ARGUMENT = 1
MAG_ERR_INVALID_ARGUMENT = 2
MAG_ERR_EMPTY_PATTERN_SET = 3
MAG_ERR_EMPTY_PATTERN = 4
MAG_ERR_BAD_CONFIG = 5
MAG_ERR_OUT_OF_RANGE = 6
MAG_ERR_NO_MEMORY = 7
MAG_ERR_INTERNAL = 8

# mag_variant (mag.h:38-44)
VARIANT_MAG, VARIANT_SMAG, VARIANT_SHIFTOR_OG, VARIANT_NAIVE, VARIANT_AC = range(5)
VARIANTS = {"mag": 0, "smag": 1, "shiftor_og": 2, "naive": 3, "ac": 4}
# mag_mapping (mag.h:46-52)
MAPPING_AUTO, MAPPING_IDENTITY, MAPPING_FREQUENCY, MAPPING_BALANCED, MAPPING_LOWBITS = -1, 0, 1, 2, 3
MAPPINGS = {"auto": -1, "identity": 0, "freq": 1, "balance": 2, "lowbits": 3}
# mag_gram_mode (mag_b200.h)
GRAM_AUTO, GRAM_EXACT, GRAM_HASHED = -1, 0, 1
# mag_scan_kernel (mag_b200.h)
KERNELS = {"auto": 0, "staged": 1, "direct": 2, "roll": 3, "pack2": 4}


class MagError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"mag status {status}: {message}")
        self.status = status
        self.message = message


class _Options(C.Structure):  # mag.h:59-70
    _fields_ = [
        ("variant", C.c_int), ("mapping", C.c_int), ("lowbits", C.c_int), ("q", C.c_int),
        ("k", C.c_int), ("sigma_prime", C.c_int), ("threads", C.c_int),
        ("histogram_sample", C.POINTER(C.c_uint8)), ("histogram_sample_len", C.c_size_t),
    ]


class _OptionsEx(C.Structure):  # mag_b200.h
    _fields_ = [
        ("base", _Options), ("gram_mode", C.c_int), ("table_bits", C.c_int),
        ("word_bits", C.c_int), ("tile_bytes", C.c_int), ("warps", C.c_int),
        ("stages", C.c_int), ("device", C.c_int), ("probes", C.c_int), ("scan_kernel", C.c_int),
        ("cluster", C.c_int),
    ]


class _Info(C.Structure):  # mag.h:82-90
    _fields_ = [
        ("variant", C.c_int), ("r", C.c_uint32), ("m", C.c_size_t), ("q", C.c_int),
        ("k", C.c_int), ("sigma_prime", C.c_int), ("mapping", C.c_int),
    ]


class _Plan(C.Structure):  # mag_b200.h mag_plan_info
    _fields_ = [
        ("variant", C.c_int), ("gram_mode", C.c_int), ("q", C.c_int), ("k", C.c_int),
        ("m_prime", C.c_int), ("sigma_prime", C.c_int), ("verify_all", C.c_int),
        ("table_bits", C.c_uint32), ("entry_bits", C.c_uint32), ("table_bytes", C.c_uint64),
        ("table_in_smem", C.c_int), ("key_len", C.c_uint32), ("prefilter_bits", C.c_uint32),
        ("bucket_bits", C.c_uint32), ("tile_bytes", C.c_uint32), ("halo", C.c_uint32),
        ("warps", C.c_uint32), ("stages", C.c_uint32), ("smem_bytes", C.c_size_t),
        ("predicted_candidates_per_byte", C.c_double), ("probes", C.c_uint32),
        ("blocks", C.c_uint32), ("direct", C.c_int), ("roll", C.c_int), ("cluster", C.c_int),
        ("pack2", C.c_int), ("measured_candidates_per_byte", C.c_double),
        ("measured_sample_bytes", C.c_uint64), ("predicted_cost", C.c_double),
        ("measured_cost", C.c_double), ("measured_plans", C.c_uint32),
        ("measured_survivors_per_byte", C.c_double), ("measured_walk_per_byte", C.c_double),
    ]


class _Metrics(C.Structure):  # mag.h:116-121
    _fields_ = [("filter_reads", C.c_uint64), ("candidates", C.c_uint64)]


class _TuneIn(C.Structure):  # mag.h:125-132
    _fields_ = [
        ("sigma", C.c_uint32), ("sigma_prime", C.c_uint32), ("r", C.c_uint64), ("m", C.c_uint64),
        ("n", C.c_uint64), ("word_bits", C.c_uint32),
    ]


class _TuneOut(C.Structure):  # mag.h:134-141
    _fields_ = [
        ("q", C.c_int), ("k", C.c_int), ("sigma_prime", C.c_int), ("rho", C.c_double),
        ("predicted_p", C.c_double), ("predicted_cost", C.c_double),
    ]


# Every symbol include/mag.h and include/mag_b200.h declare.
EXPORTS = [
    "mag_options_init", "mag_engine_create", "mag_engine_destroy", "mag_engine_get_info",
    "mag_engine_copy_alphabet", "mag_prepare_text", "mag_prepared_destroy",
    "mag_search_prepared", "mag_search", "mag_matches_count", "mag_matches_get",
    "mag_matches_metrics", "mag_matches_destroy", "mag_tune", "mag_sample_patterns",
    "mag_patterns_count", "mag_patterns_get", "mag_patterns_destroy", "mag_status_string",
    "mag_last_error", "mag_version",
    # mag_b200.h
    "mag_options_ex_init", "mag_engine_create_ex", "mag_engine_get_plan",
    "mag_prepare_device_text", "mag_search_prepared_async", "mag_matches_sync",
    "mag_matches_copy", "mag_prepared_copy_codes", "mag_engine_copy_masks",
    "mag_kernel_launches", "mag_scan_timer_enable", "mag_scan_timer_read",
]

_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Loads the in-tree libmag_b200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, sz, st = C.c_void_p, C.c_size_t, C.c_int
    u8p = C.POINTER(C.c_uint8)
    sig = {
        "mag_options_init": (None, [C.POINTER(_Options)]),
        "mag_options_ex_init": (None, [C.POINTER(_OptionsEx)]),
        "mag_engine_create": (st, [C.POINTER(u8p), C.POINTER(sz), sz, C.POINTER(_Options), C.POINTER(vp)]),
        "mag_engine_create_ex": (st, [C.POINTER(u8p), C.POINTER(sz), sz, C.POINTER(_OptionsEx), C.POINTER(vp)]),
        "mag_engine_destroy": (None, [vp]),
        "mag_engine_get_info": (st, [vp, C.POINTER(_Info)]),
        "mag_engine_get_plan": (st, [vp, C.POINTER(_Plan)]),
        "mag_engine_copy_alphabet": (st, [vp, u8p, C.POINTER(C.c_uint32)]),
        "mag_engine_copy_masks": (st, [vp, C.POINTER(C.c_uint64), sz]),
        "mag_prepare_text": (st, [vp, vp, sz, C.POINTER(vp)]),
        "mag_prepare_device_text": (st, [vp, vp, sz, C.POINTER(vp)]),
        "mag_prepared_destroy": (None, [vp]),
        "mag_prepared_copy_codes": (st, [vp, C.POINTER(C.c_uint32), sz]),
        "mag_search_prepared": (st, [vp, vp, C.POINTER(vp)]),
        "mag_search_prepared_async": (st, [vp, vp, vp, C.POINTER(vp)]),
        "mag_search": (st, [vp, vp, sz, C.POINTER(vp)]),
        "mag_matches_count": (sz, [vp]),
        "mag_matches_get": (st, [vp, sz, C.POINTER(C.c_uint32), C.POINTER(sz)]),
        "mag_matches_copy": (st, [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), sz]),
        "mag_matches_metrics": (st, [vp, C.POINTER(_Metrics)]),
        "mag_matches_sync": (st, [vp]),
        "mag_matches_destroy": (None, [vp]),
        "mag_tune": (st, [C.POINTER(_TuneIn), C.POINTER(_TuneOut)]),
        "mag_sample_patterns": (st, [vp, sz, sz, sz, C.c_uint64, C.POINTER(vp)]),
        "mag_patterns_count": (sz, [vp]),
        "mag_patterns_get": (st, [vp, sz, C.POINTER(u8p), C.POINTER(sz)]),
        "mag_patterns_destroy": (None, [vp]),
        "mag_status_string": (C.c_char_p, [st]),
        "mag_last_error": (C.c_char_p, []),
        "mag_version": (C.c_char_p, []),
        "mag_kernel_launches": (C.c_uint64, []),
        "mag_scan_timer_enable": (None, [C.c_int]),
        "mag_scan_timer_read": (st, [C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(status: int) -> None:
    if status != MAG_OK:
        L = lib()
        raise MagError(status, L.mag_last_error().decode(errors="replace"))


def _as_u8(buf) -> np.ndarray:
    if isinstance(buf, np.ndarray):
        a = np.ascontiguousarray(buf.view(np.uint8).reshape(-1))
    else:
        a = np.frombuffer(bytes(buf), dtype=np.uint8)
    return a


def _u8ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


@dataclass
class EngineInfo:
    variant: int
    r: int
    m: int
    q: int
    k: int
    sigma_prime: int
    mapping: int


@dataclass
class Metrics:
    filter_reads: int
    candidates: int


class Matches:
    """Sorted (offset, pattern_index) occurrences (mag.h:111-122).

    A pending (asynchronous) handle keeps the prepared text it searches
    alive until it is closed: materialising may search that text again
    (staging overflow), so the device text must outlive it (mag_b200.h).
    """

    def __init__(self, handle: int, keep=None):
        self._h = C.c_void_p(handle)
        self._keep = keep

    def __len__(self) -> int:
        return int(lib().mag_matches_count(self._h))

    def get(self, index: int):
        pid, off = C.c_uint32(), C.c_size_t()
        _check(lib().mag_matches_get(self._h, index, C.byref(pid), C.byref(off)))
        return int(off.value), int(pid.value)

    def arrays(self):
        """(offsets uint64[n], pattern_indices uint32[n]) in canonical order."""
        n = len(self)
        offs = np.empty(n, dtype=np.uint64)
        pids = np.empty(n, dtype=np.uint32)
        _check(lib().mag_matches_copy(self._h, offs.ctypes.data_as(C.POINTER(C.c_uint64)),
                                      pids.ctypes.data_as(C.POINTER(C.c_uint32)), n))
        return offs, pids

    def pairs(self):
        offs, pids = self.arrays()
        return list(zip(offs.tolist(), pids.tolist()))

    def metrics(self) -> Metrics:
        m = _Metrics()
        _check(lib().mag_matches_metrics(self._h, C.byref(m)))
        return Metrics(int(m.filter_reads), int(m.candidates))

    def sync(self) -> None:
        _check(lib().mag_matches_sync(self._h))

    def close(self) -> None:
        if self._h:
            lib().mag_matches_destroy(self._h)
            self._h = C.c_void_p()
        self._keep = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Prepared:
    """Text prepared for an engine (mag.h:98-102).  Keeps the host buffer alive."""

    def __init__(self, handle: int, keep):
        self._h = C.c_void_p(handle)
        self._keep = keep

    def codes(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint32)
        _check(lib().mag_prepared_copy_codes(self._h, out.ctypes.data_as(C.POINTER(C.c_uint32)), count))
        return out

    def close(self) -> None:
        if self._h:
            lib().mag_prepared_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    """A compiled pattern set (mag_engine_create, mag.h:75-80).

    Keyword options mirror ``mag_options`` (variant, mapping, lowbits, q, k,
    sigma_prime, threads, histogram_sample) plus the GPU extras of
    ``mag_options_ex`` (gram_mode, table_bits, word_bits, tile_bytes, warps,
    stages, device, probes, scan_kernel; device=-2 builds the host tables
    only, no upload).  ``histogram_sample`` of >= 4 KiB of text also lets the
    planner measure its finalist plans' candidate rates on it.
    """

    def __init__(self, patterns: Sequence[bytes], variant="mag", mapping="auto", lowbits=0, q=0, k=0,
                 sigma_prime=0, threads=1, histogram_sample: Optional[bytes] = None,
                 gram_mode=GRAM_AUTO, table_bits=0, word_bits=0, tile_bytes=0, warps=0, stages=0,
                 device=-1, probes=0, scan_kernel="auto", cluster=0):
        L = lib()
        self._h = C.c_void_p()
        opts = _OptionsEx()
        L.mag_options_ex_init(C.byref(opts))
        opts.base.variant = VARIANTS[variant] if isinstance(variant, str) else int(variant)
        opts.base.mapping = MAPPINGS[mapping] if isinstance(mapping, str) else int(mapping)
        opts.base.lowbits, opts.base.q, opts.base.k = int(lowbits), int(q), int(k)
        opts.base.sigma_prime, opts.base.threads = int(sigma_prime), int(threads)
        self._sample = None
        if histogram_sample is not None:
            self._sample = _as_u8(histogram_sample)
            opts.base.histogram_sample = _u8ptr(self._sample)
            opts.base.histogram_sample_len = self._sample.size
        opts.gram_mode, opts.table_bits, opts.word_bits = int(gram_mode), int(table_bits), int(word_bits)
        opts.tile_bytes, opts.warps, opts.stages, opts.device = int(tile_bytes), int(warps), int(stages), int(device)
        opts.probes = int(probes)
        opts.scan_kernel = KERNELS[scan_kernel] if isinstance(scan_kernel, str) else int(scan_kernel)
        opts.cluster = int(cluster)
        bufs = [_as_u8(p) for p in patterns]
        n = len(bufs)
        ptrs = (C.POINTER(C.c_uint8) * max(n, 1))(*[_u8ptr(b) for b in bufs])
        lens = (C.c_size_t * max(n, 1))(*[b.size for b in bufs])
        _check(L.mag_engine_create_ex(ptrs, lens, n, C.byref(opts), C.byref(self._h)))

    # -- introspection
    def info(self) -> EngineInfo:
        i = _Info()
        _check(lib().mag_engine_get_info(self._h, C.byref(i)))
        return EngineInfo(i.variant, i.r, i.m, i.q, i.k, i.sigma_prime, i.mapping)

    def plan(self) -> dict:
        p = _Plan()
        _check(lib().mag_engine_get_plan(self._h, C.byref(p)))
        return {f: getattr(p, f) for f, _ in _Plan._fields_}

    def alphabet(self):
        t = (C.c_uint8 * 256)()
        sp = C.c_uint32()
        _check(lib().mag_engine_copy_alphabet(self._h, t, C.byref(sp)))
        return bytes(t), int(sp.value)

    def masks(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        _check(lib().mag_engine_copy_masks(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)), count))
        return out

    # -- search
    def prepare(self, text) -> Prepared:
        a = _as_u8(text)
        h = C.c_void_p()
        _check(lib().mag_prepare_text(self._h, a.ctypes.data_as(C.c_void_p), a.size, C.byref(h)))
        return Prepared(h.value, a)

    def prepare_device(self, ptr: int, length: int, keep=None) -> Prepared:
        h = C.c_void_p()
        _check(lib().mag_prepare_device_text(self._h, C.c_void_p(ptr), length, C.byref(h)))
        return Prepared(h.value, keep)

    def search_prepared(self, prepared: Prepared) -> Matches:
        h = C.c_void_p()
        _check(lib().mag_search_prepared(self._h, prepared._h, C.byref(h)))
        return Matches(h.value, keep=prepared)

    def search_prepared_async(self, prepared: Prepared, stream: int = 0) -> Matches:
        h = C.c_void_p()
        _check(lib().mag_search_prepared_async(self._h, prepared._h, C.c_void_p(stream), C.byref(h)))
        return Matches(h.value, keep=prepared)

    def search(self, text) -> Matches:
        """prepare + search (mag_search): host text in, sorted matches out."""
        if isinstance(text, np.ndarray) and text.dtype == np.uint8 and text.flags.c_contiguous:
            a = text
        else:
            a = _as_u8(text)
        h = C.c_void_p()
        _check(lib().mag_search(self._h, a.ctypes.data_as(C.c_void_p), a.size, C.byref(h)))
        return Matches(h.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().mag_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tune(sigma: int, r: int, m: int, n: int = 1 << 20, sigma_prime: int = 0, word_bits: int = 0) -> dict:
    """mag_tune (mag.h:124-143): the reference's parameter rule, restated."""
    ti = _TuneIn(sigma, sigma_prime, r, m, n, word_bits)
    to = _TuneOut()
    _check(lib().mag_tune(C.byref(ti), C.byref(to)))
    return {f: getattr(to, f) for f, _ in _TuneOut._fields_}


def sample_patterns(corpus, count: int, length: int, seed: int):
    """mag_sample_patterns (mag.h:145-153): seeded substrings of the corpus."""
    a = _as_u8(corpus)
    h = C.c_void_p()
    L = lib()
    _check(L.mag_sample_patterns(a.ctypes.data_as(C.c_void_p), a.size, count, length, seed, C.byref(h)))
    try:
        out = []
        for i in range(L.mag_patterns_count(h)):
            p, ln = C.POINTER(C.c_uint8)(), C.c_size_t()
            _check(L.mag_patterns_get(h, i, C.byref(p), C.byref(ln)))
            out.append(C.string_at(p, ln.value))
        return out
    finally:
        L.mag_patterns_destroy(h)


def status_string(status: int) -> str:
    return lib().mag_status_string(status).decode()


def version() -> str:
    return lib().mag_version().decode()


def scan_timer(enable, scan_only: bool = False) -> None:
    """Bracket every search's kernels with CUDA events (bench/profiling):
    the scan kernel + finish grid, or with scan_only the scan kernel alone."""
    lib().mag_scan_timer_enable((2 if scan_only else 1) if enable else 0)


def scan_timer_read():
    """(total device ms, launches) of the timed scan kernels so far."""
    ms, n = C.c_double(), C.c_uint64()
    _check(lib().mag_scan_timer_read(C.byref(ms), C.byref(n)))
    return float(ms.value), int(n.value)


def kernel_launches() -> int:
    return int(lib().mag_kernel_launches())
