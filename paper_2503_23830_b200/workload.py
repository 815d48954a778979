"""Synthetic multimodal batches of the BASELINE configs (host-side input
generation for bench.py / tests; not part of the dispatch path).

`generate` restates the reference's deterministic MCI generator
(proj/src/workload.cpp:20-161: std::mt19937_64, Box-Muller normals, Gaussian
copula between two modalities, log-normal / uniform / fixed lengths with
clipping), so the same seed gives the reference's exact examples; this is
checked against the reference library in tests/test_workload.py. Profiles
and weights are SURVEY.md section 8(d).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the C++ standard's parameters)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & MASK64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


class _Rng:  # workload.cpp:22-37
    def __init__(self, seed):
        self.e = MT19937_64(seed)

    def uniform01(self):
        return ((self.e() >> 11) + 0.5) * 2.0 ** -53

    def normal(self):
        u1 = self.uniform01()
        u2 = self.uniform01()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


@dataclass
class LengthDist:
    kind: str = "fixed"  # "lognormal" | "uniform" | "fixed"
    mu: float = 0.0
    sigma: float = 1.0
    lo: int = 1
    hi: int = 1
    clip_min: int = 1
    clip_max: int = 0


@dataclass
class TaskProfile:
    name: str
    parts: list  # [(modality, LengthDist)]
    correlation: float = 0.0
    correlated_a: str = ""
    correlated_b: str = ""


def _sample_length(dist: LengthDist, z: float) -> int:  # workload.cpp:41-60
    if dist.kind == "fixed":
        ln = dist.lo
    elif dist.kind == "uniform":
        u = 0.5 * math.erfc(-z / math.sqrt(2.0))
        ln = dist.lo + int(u * float(dist.hi - dist.lo + 1))
        ln = min(ln, dist.hi)
    else:
        ln = int(math.ceil(math.exp(dist.mu + dist.sigma * z)))
    if dist.clip_max > 0:
        ln = min(ln, dist.clip_max)
    return max(ln, dist.clip_min, 1)


@dataclass
class Example:
    example_id: int
    modality: list = field(default_factory=list)
    meta: list = field(default_factory=list)


def generate(profiles, weights, n: int, seed: int):
    """workload.cpp:107-161."""
    rng = _Rng(seed)
    out = []
    for ex_id in range(n):
        pick = rng.uniform01()
        chosen = len(profiles) - 1
        cum = 0.0
        for p, w in enumerate(weights):
            cum += w
            if pick < cum:
                chosen = p
                break
        prof = profiles[chosen]
        z_shared = rng.normal() if prof.correlation != 0.0 else 0.0
        ex = Example(ex_id)
        for modality, dist in prof.parts:
            z = rng.normal()
            if prof.correlation != 0.0:
                if modality == prof.correlated_a:
                    z = z_shared
                elif modality == prof.correlated_b:
                    rho = prof.correlation
                    z = rho * z_shared + math.sqrt(1.0 - rho * rho) * z
            ex.modality.append(modality)
            ex.meta.append(_sample_length(dist, z))
        out.append(ex)
    return out


def _ln(mu, sigma, lo, hi):
    return LengthDist("lognormal", mu, sigma, clip_min=lo, clip_max=hi)


VISION_INSTRUCT = TaskProfile("vision-instruct", [("vision", _ln(6.5, 0.8, 64, 4096)),
                                                  ("text", _ln(5.0, 1.0, 8, 2048))])
TEXT_ONLY = TaskProfile("text-only", [("text", _ln(6.0, 1.0, 16, 8192))])
ASR = TaskProfile("asr", [("audio", _ln(6.8, 0.6, 50, 3000)), ("text", _ln(4.0, 0.6, 4, 512))],
                  0.9, "audio", "text")
SPEECH_QA = TaskProfile("speech-qa", [("audio", _ln(6.5, 0.7, 50, 3000)),
                                      ("text", _ln(3.0, 1.2, 2, 1024))])

MIXES = {
    2: ([VISION_INSTRUCT, TEXT_ONLY], [0.6, 0.4]),                       # C2
    3: ([VISION_INSTRUCT, ASR, SPEECH_QA, TEXT_ONLY], [0.4, 0.2, 0.2, 0.2]),  # C3 / C4
}
MODALITY_CODE = {"text": 0, "vision": 1, "audio": 2}


@dataclass
class Batch:
    """One global batch in flat arrays (example order = reference input order)."""
    d: int
    origin: np.ndarray        # [E] int32, round-robin j % d (simulate.cpp:41)
    part_offset: np.ndarray   # [E+1] int32
    modality: np.ndarray      # [parts] int32 codes
    meta: np.ndarray          # [parts] int64 metadata lengths
    rates: np.ndarray         # [3] downsample rate per modality code
    encoded: np.ndarray       # [parts] ceil(meta / rate)
    interleaved: np.ndarray   # [E] sum of encoded parts

    def phase_items(self, modality: str):
        """Encoder phase universe (orchestrator.cpp:247-267): the parts of that
        modality in example order, metadata lengths, the example's origin."""
        code = MODALITY_CODE[modality]
        idx = np.nonzero(self.modality == code)[0]
        ex = np.searchsorted(self.part_offset, idx, side="right") - 1
        return self.meta[idx].astype(np.int64), self.origin[ex].astype(np.int32), idx

    def llm_items(self):
        """Backbone universe (orchestrator.cpp:421-426): whole examples, length
        = interleaved length of the encoded parts."""
        return self.interleaved.astype(np.int64), self.origin.astype(np.int32)


def make_batch(mix: int, d: int, per_instance: int, seed: int,
               rates=(1, 4, 4)) -> Batch:
    profiles, weights = MIXES[mix]
    E = d * per_instance
    exs = generate(profiles, weights, E, seed)
    po = np.zeros(E + 1, np.int32)
    mod, meta = [], []
    for j, ex in enumerate(exs):
        po[j + 1] = po[j] + len(ex.meta)
        mod += [MODALITY_CODE[m] for m in ex.modality]
        meta += ex.meta
    mod = np.asarray(mod, np.int32)
    meta = np.asarray(meta, np.int64)
    r = np.asarray(rates, np.int64)
    enc = (meta + r[mod] - 1) // r[mod]
    inter = np.add.reduceat(enc, po[:-1]) if E else np.zeros(0, np.int64)
    origin = (np.arange(E) % d).astype(np.int32)
    return Batch(d, origin, po, mod, meta, r, enc, inter.astype(np.int64))
