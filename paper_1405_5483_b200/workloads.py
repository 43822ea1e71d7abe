"""Seeded synthetic stand-ins for the five BASELINE.json configurations.

The reference benchmarks on Pizza&Chili corpora, which
are not available offline; these generators reproduce the shapes, sizes and
value distributions BASELINE.json names.  Everything is
numpy with fixed seeds, so a (config, scale) pair always yields the same
bytes.  Pattern order is fixed: the copied half first, then the generated
half.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np

DNA = np.frombuffer(b"ACGT", dtype=np.uint8)
PROTEIN = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", dtype=np.uint8)
# space + 63 letters for the English-like config
ENGLISH = np.frombuffer(b"etaoinshrdlcumwfgypbvkjxqzETAOINSHRDLCUMWFGYPBVKJXQZ0123456789-", dtype=np.uint8)


@dataclass
class Workload:
    name: str
    text: np.ndarray  # uint8
    patterns: List[bytes]
    meta: dict = field(default_factory=dict)


def _zipf_probs(k: int, s: float) -> np.ndarray:
    w = 1.0 / np.arange(1, k + 1, dtype=np.float64) ** s
    return w / w.sum()


def _iid(rng, alphabet: np.ndarray, n: int, probs=None) -> np.ndarray:
    if probs is None:
        idx = rng.integers(0, alphabet.size, size=n, dtype=np.uint8)
    else:
        idx = rng.choice(alphabet.size, size=n, p=probs).astype(np.uint8)
    return alphabet[idx]


def _english(rng, n: int) -> np.ndarray:
    """Zipf(1.0) letters; a space after geometric(mean 5, support >= 1) words."""
    letters = _iid(rng, ENGLISH, n, _zipf_probs(ENGLISH.size, 1.0))
    # word lengths until the text is covered
    est = n // 6 + 64
    lens = rng.geometric(0.2, size=est)
    while (lens + 1).sum() < n:
        lens = np.concatenate([lens, rng.geometric(0.2, size=est)])
    ends = np.cumsum(lens + 1) - 1
    ends = ends[ends < n]
    letters[ends] = ord(" ")
    return letters


def _copied(rng, text: np.ndarray, count: int, m: int) -> List[bytes]:
    offs = rng.integers(0, text.size - m + 1, size=count)
    return [text[o:o + m].tobytes() for o in offs]


def generate(cfg: int, scale: float = 1.0, seed: int = 0) -> Workload:
    """Config cfg (1..5) at `scale` of its full text size (patterns unchanged
    unless the text gets too small for them)."""
    rng = np.random.default_rng(1405_5483 + 1000 * cfg + seed)
    if cfg == 1:
        n, r, m = 16 << 20, 100, 16
        text = _iid(rng, DNA, max(int(n * scale), 64))
        pats = _copied(rng, text, r // 2, m) + [_iid(rng, DNA, m).tobytes() for _ in range(r - r // 2)]
        return Workload("cfg1-dna-16MiB-r100-m16", text, pats, dict(n=n, r=r, m=m, sigma=4))
    if cfg == 2:
        n, r, m = 1 << 30, 10_000, 32
        text = _iid(rng, DNA, max(int(n * scale), 64))
        gen = _iid(rng, DNA, (r - r // 2) * m).reshape(-1, m)
        pats = _copied(rng, text, r // 2, m) + [row.tobytes() for row in gen]
        return Workload("cfg2-dna-1GiB-r10k-m32", text, pats, dict(n=n, r=r, m=m, sigma=4))
    if cfg == 3:
        n, r, m = 256 << 20, 1000, 16
        probs = _zipf_probs(PROTEIN.size, 0.7)
        text = _iid(rng, PROTEIN, max(int(n * scale), 64), probs)
        gen = _iid(rng, PROTEIN, (r - r // 2) * m, probs).reshape(-1, m)
        pats = _copied(rng, text, r // 2, m) + [row.tobytes() for row in gen]
        return Workload("cfg3-protein-zipf0.7-256MiB-r1k-m16", text, pats, dict(n=n, r=r, m=m, sigma=20))
    if cfg == 4:
        n, r, m = 512 << 20, 100_000, 32
        text = _english(rng, max(int(n * scale), 4096))
        gen_src = _english(rng, (r - r // 2) * m * 2 + 1024)
        starts = rng.integers(0, gen_src.size - m + 1, size=r - r // 2)
        pats = _copied(rng, text, r // 2, m) + [gen_src[s:s + m].tobytes() for s in starts]
        return Workload("cfg4-english-zipf1-512MiB-r100k-m32", text, pats, dict(n=n, r=r, m=m, sigma=64))
    if cfg == 5:
        n, r, m = 1 << 30, 100_000, 12
        nn = max(int(n * scale), 4096)
        text = _iid(rng, DNA, nn)
        pats_arr = _iid(rng, DNA, r * m).reshape(r, m)
        plants = int(0.01 * nn)
        done = 0
        ar = np.arange(m)
        while done < plants:  # generation order: later plants overwrite earlier ones
            b = min(1 << 20, plants - done)
            offs = rng.integers(0, nn - m + 1, size=b)
            ids = rng.integers(0, r, size=b)
            text[(offs[:, None] + ar).reshape(-1)] = pats_arr[ids].reshape(-1)
            done += b
        pats = [row.tobytes() for row in pats_arr]
        return Workload("cfg5-dna-1GiB-r100k-m12-planted1pct", text, pats,
                        dict(n=n, r=r, m=m, sigma=4, plants=plants))
    raise ValueError(f"unknown config {cfg}")


CONFIGS = {1: "cfg1", 2: "cfg2", 3: "cfg3", 4: "cfg4", 5: "cfg5"}
