"""Seeded synthetic inputs for the five BASELINE.json configs (C1-C5).

The reference publishes no benchmark suite for this path; these generators
stand in with the shapes, sizes and value distributions BASELINE.json states
(SURVEY.md §8d). Seeds follow the reference bench default (bench.hpp:19,
seed 2018) + config index; series B of C3 uses seed + 100. The bit generator
is numpy's MT19937 (the Mersenne-Twister family the reference names for its
generators, dataset.hpp:36-37). Series are generated once on the host in
fp64 and fed byte-identically to the GPU and to the CPU oracle.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

BASE_SEED = 2018
BEAT_SIGMA = 8.0  # C4 beat width (samples); BASELINE leaves it open


@dataclass
class Config:
    name: str
    a: np.ndarray
    b: Optional[np.ndarray]
    window: int
    ez: float
    description: str
    planted: Optional[dict] = None

    @property
    def self_join(self) -> bool:
        return self.b is None

    @property
    def zone(self) -> int:
        return 0 if self.b is not None else int(np.floor(self.window * self.ez + 0.5))

    def cells(self) -> int:
        La = self.a.size - self.window + 1
        if self.b is not None:
            return La * (self.b.size - self.window + 1)
        r = La - self.zone - 1
        return r * (r + 1) // 2 if r > 0 else 0


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.MT19937(seed))


def random_walk(n: int, seed: int) -> np.ndarray:
    """Gaussian random walk: cumulative sum of N(0,1) increments."""
    return np.cumsum(rng(seed).standard_normal(n))


def checksum(x: np.ndarray) -> str:
    """Workload checksum of a series (series_checksum, bench.hpp:39-42; the
    reference declares it without a body): BLAKE2b-64 over all fp64 bytes,
    plus the length. Both bench arms print it, so a reader can check that they
    timed the same input."""
    import hashlib
    h = hashlib.blake2b(np.ascontiguousarray(x, dtype=np.float64).tobytes(), digest_size=8)
    return f"{h.hexdigest()}-{x.size}"


def _starts(g: np.random.Generator, n: int, count: int, length: int, sep: int) -> np.ndarray:
    """`count` seeded non-overlapping segment starts, pairwise gaps > sep."""
    for _ in range(10000):
        s = np.sort(g.integers(0, n - length, size=count))
        if count < 2 or np.all(np.diff(s) > length + sep):
            return g.permutation(s)
    raise RuntimeError("could not place segments")


def c1(n: int = 16384, m: int = 256) -> Config:
    return Config("C1", random_walk(n, BASE_SEED + 1), None, m, 0.5,
                  f"self-join random walk n={n} m={m}")


def c2(n: int = 131072, m: int = 1024) -> Config:
    """Random walk + 3 planted motif pairs (segment replacement) + 1 discord."""
    g = rng(BASE_SEED + 2)
    x = np.cumsum(g.standard_normal(n))
    st = _starts(g, n, 7, m, m)
    t = np.arange(m)
    pairs = []
    for p in range(3):
        f = g.uniform(1.0, 8.0)
        burst = 5.0 * np.sin(2.0 * np.pi * f * t / m)
        s1, s2 = int(st[2 * p]), int(st[2 * p + 1])
        for s in (s1, s2):
            x[s:s + m] = x[s] + burst + g.normal(0.0, 0.1, m)
        pairs.append((s1, s2, f))
    sd = int(st[6])
    x[sd:sd + m] = x[sd] + g.uniform(-5.0, 5.0, m)
    return Config("C2", x, None, m, 0.5, f"self-join walk+motifs n={n} m={m}",
                  planted={"pairs": pairs, "discord": sd})


def c3(na: int = 262144, nb: int = 65536, m: int = 512) -> Config:
    return Config("C3", random_walk(na, BASE_SEED + 3), random_walk(nb, BASE_SEED + 3 + 100), m, 0.0,
                  f"AB-join walks n_a={na} n_b={nb} m={m}")


def c4(n: int = 1 << 20, m: int = 256) -> Config:
    """ECG-like: Gaussian beats, baseline wander, noise, two constant segments."""
    g = rng(BASE_SEED + 4)
    centers = [float(g.uniform(0, 280))]
    while centers[-1] < n + 300:
        centers.append(centers[-1] + g.uniform(200.0, 280.0))
    centers = np.asarray(centers)
    amps = g.uniform(0.8, 1.2, centers.size)
    t = np.arange(n, dtype=np.float64)
    k = np.clip(np.searchsorted(centers, t), 1, centers.size - 1)
    x = np.zeros(n)
    for kk in (k - 1, k):  # beats are >= 200 apart, sigma 8: two nearest suffice
        x += amps[kk] * np.exp(-0.5 * ((t - centers[kk]) / BEAT_SIGMA) ** 2)
    x += 0.2 * np.sin(2.0 * np.pi * t / 50000.0)
    x += g.normal(0.0, 0.05, n)
    flats = _starts(g, n, 2, 5000, m)
    for s in flats:
        s = int(s)
        x[s:s + 5000] = x[s]
    return Config("C4", x, None, m, 0.5, f"self-join ECG-like n={n} m={m}",
                  planted={"flat_segments": [int(s) for s in flats]})


def c5(n: int = 1 << 23, m: int = 128) -> Config:
    return Config("C5", random_walk(n, BASE_SEED + 5), None, m, 0.5,
                  f"self-join random walk n={n} m={m}")


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def get(name: str, **kw) -> Config:
    return CONFIGS[name.upper()](**kw)
