"""Seeded synthetic top-K retrieval workloads (shared by tests, bench and smoke).

This module only *draws inputs*. It holds none of the method's arithmetic (no
Eq. 1, no overlap counting, no clustering); both the CUDA path and the CPU
oracle consume its arrays unchanged.

Recipe (restated in DESIGN.md "Input recipe"):

* ``numpy.random.Generator(PCG64(seed))``.
* ``perm = rng.permutation(V)`` maps popularity rank r to DocId, decorrelating
  popularity from the ID value.
* Popularity weights ``w_r ∝ (r+1)^(-s_zipf)`` ("79.2% / 57.4% /
  49.6% of questions draw from the top 20% most frequently accessed documents";
  s_zipf = 0.8 lands the top-20% slot share inside that band).
* Single turn: T = ceil(N/g) topics; each topic core is K distinct ranks drawn
  ∝ w.  Context i belongs to topic i // g and takes round(ω·K) ranks uniformly
  from its core; the remaining K − round(ω·K) distinct ranks are drawn ∝ w,
  rejecting repeats.  Retrieval order is a uniform permutation of the K docs.
  Rows are finally shuffled so topic-mates are not adjacent.
* Multi-turn: ceil(N/turns) sessions; turn 0 as above; turn t ≥ 1 draws
  round(τ·K) docs uniformly from the session's history ("40% of
  retrieved documents in any turn overlap with earlier ones in the same
  session") and fills the rest ∝ w excluding the history.
* Edge inputs: all-disjoint, all-identical, all-permutations-of-one-set.

Variable lengths (``len_min`` < K) fill slots past ``lens[i]`` with junk IDs
that the consumer must ignore.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

PAD_ID = np.uint32(0xFFFFFFFF)  # never a valid DocId (include/ragb.h)


@dataclasses.dataclass
class Workload:
    ids: np.ndarray            # uint32 [N, K], row-major, retrieval order
    lens: np.ndarray | None    # uint8 [N] or None (all K)
    session: np.ndarray | None  # int64 [N] (multi-turn only)
    turn: np.ndarray | None     # int64 [N] (multi-turn only)
    recipe: dict

    @property
    def N(self) -> int:
        return int(self.ids.shape[0])

    @property
    def K(self) -> int:
        return int(self.ids.shape[1])


# Config table of SURVEY.md §8(d) / BASELINE.json "configs".
CONFIGS = {
    "C1": dict(N=64, K=5, V=200, seed=1),
    "C2": dict(N=4096, K=10, V=20_000, seed=2),
    "C3": dict(N=32_768, K=15, V=200_000, seed=3, turns=5),
    "C4": dict(N=100_000, K=20, V=1_000_000, seed=4),
    "C5": dict(N=16_384, K=20, V=200_000, seed=5),  # K is swept 5..100
}


class _Sampler:
    """Inverse-CDF sampler over popularity ranks, w_r ∝ (r+1)^-s."""

    def __init__(self, rng: np.random.Generator, V: int, s_zipf: float):
        self.rng = rng
        w = (np.arange(1, V + 1, dtype=np.float64)) ** (-s_zipf)
        c = np.cumsum(w)
        self.cdf = c / c[-1]
        self.V = V

    def draw(self, shape) -> np.ndarray:
        u = self.rng.random(shape)
        r = np.searchsorted(self.cdf, u, side="right")
        return np.minimum(r, self.V - 1).astype(np.int64)

    def distinct_rows(self, n_rows: int, need: int, exclude: list[np.ndarray] | None = None) -> np.ndarray:
        """For each row, `need` distinct ranks drawn ∝ w (rejecting repeats and `exclude[row]`)."""
        out = np.empty((n_rows, need), dtype=np.int64)
        if need == 0:
            return out
        batch = self.draw((n_rows, 2 * need + 8))
        for i in range(n_rows):
            seen = set() if exclude is None else set(exclude[i].tolist())
            got = 0
            cand = batch[i]
            pos = 0
            while got < need:
                if pos == cand.shape[0]:
                    cand = self.draw(2 * need + 8)
                    pos = 0
                r = int(cand[pos])
                pos += 1
                if r not in seen:
                    seen.add(r)
                    out[i, got] = r
                    got += 1
        return out


def _row_shuffle(rng: np.random.Generator, a: np.ndarray) -> np.ndarray:
    keys = rng.random(a.shape)
    idx = np.argsort(keys, axis=1, kind="stable")
    return np.take_along_axis(a, idx, axis=1)


def _single_turn_ranks(rng, smp: _Sampler, N: int, K: int, g: int, omega: float) -> np.ndarray:
    T = math.ceil(N / g)
    cores = smp.distinct_rows(T, K)
    q = int(round(omega * K))
    topic = np.arange(N) // g
    # round(ω·K) ranks uniformly (without replacement) from the topic core.
    pick = np.argsort(rng.random((N, K)), axis=1)[:, :q]
    core_part = np.take_along_axis(cores[topic], pick, axis=1)
    bg = smp.distinct_rows(N, K - q, exclude=list(core_part))
    ranks = np.concatenate([core_part, bg], axis=1)
    return _row_shuffle(rng, ranks)  # retrieval order = uniform permutation


def generate(N: int, K: int, V: int, seed: int, *, s_zipf: float = 0.8, g: int = 8,
             omega: float = 0.4, turns: int = 1, tau: float = 0.4,
             len_min: int | None = None) -> Workload:
    """Draw one workload. ``turns > 1`` gives multi-turn sessions."""
    if not (1 <= K <= 255):
        raise ValueError("K must be in [1, 255]")
    if K > V:
        raise ValueError("K > V: cannot draw K distinct docs")
    rng = np.random.Generator(np.random.PCG64(seed))
    perm = rng.permutation(V).astype(np.uint32)
    smp = _Sampler(rng, V, s_zipf)
    if turns <= 1:
        ranks = _single_turn_ranks(rng, smp, N, K, g, omega)
        ranks = ranks[rng.permutation(N)]
        session = turn = None
    else:
        S = math.ceil(N / turns)
        t0 = _single_turn_ranks(rng, smp, S, K, g, omega)
        rows = [t0]
        hist = [set(r.tolist()) for r in t0]
        qk = int(round(tau * K))
        for _t in range(1, turns):
            cur = np.empty((S, K), dtype=np.int64)
            for s in range(S):
                h = np.fromiter(hist[s], dtype=np.int64)
                h.sort()
                qq = min(qk, h.shape[0])
                old = rng.choice(h, size=qq, replace=False)
                cur[s, :qq] = old
            new = smp.distinct_rows(S, K - min(qk, K), exclude=[np.fromiter(h_, dtype=np.int64) for h_ in hist])
            cur[:, min(qk, K):] = new
            cur = _row_shuffle(rng, cur)
            for s in range(S):
                hist[s].update(cur[s].tolist())
            rows.append(cur)
        allr = np.stack(rows, axis=1).reshape(S * turns, K)  # session-major
        sess = np.repeat(np.arange(S), turns)
        trn = np.tile(np.arange(turns), S)
        allr, sess, trn = allr[:N], sess[:N], trn[:N]
        order = rng.permutation(N)
        ranks, session, turn = allr[order], sess[order].astype(np.int64), trn[order].astype(np.int64)
    ids = perm[ranks].astype(np.uint32)
    lens = None
    if len_min is not None and len_min < K:
        lens = rng.integers(len_min, K + 1, size=N).astype(np.uint8)
        junk = rng.integers(0, 2**32 - 1, size=ids.shape, dtype=np.uint64).astype(np.uint32)
        col = np.arange(K)[None, :]
        ids = np.where(col < lens[:, None].astype(np.int64), ids, junk).astype(np.uint32)
    recipe = dict(N=N, K=K, V=V, seed=seed, s_zipf=s_zipf, g=g, omega=omega, turns=turns,
                  tau=tau, len_min=len_min)
    return Workload(np.ascontiguousarray(ids), lens, session, turn, recipe)


def config(name: str, **over) -> Workload:
    kw = dict(CONFIGS[name])
    kw.update(over)
    return generate(**kw)


def edge(kind: str, N: int, K: int, seed: int = 0) -> Workload:
    """Degenerate inputs of SURVEY.md §8(d) "Edge" row."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "disjoint":
        ids = np.arange(N * K, dtype=np.uint32).reshape(N, K)
    elif kind == "identical":
        row = rng.permutation(10 * K + 10)[:K].astype(np.uint32)
        ids = np.tile(row, (N, 1))
    elif kind == "permutations":
        row = rng.permutation(10 * K + 10)[:K].astype(np.uint32)
        ids = _row_shuffle(rng, np.tile(row, (N, 1))).astype(np.uint32)
    else:
        raise ValueError(kind)
    return Workload(np.ascontiguousarray(ids), None, None, None, dict(kind=kind, N=N, K=K, seed=seed))


def top20_slot_share(ids: np.ndarray, lens: np.ndarray | None = None) -> float:
    """Share of retrieval slots filled by the 20% most-retrieved distinct docs."""
    if lens is None:
        flat = ids.reshape(-1)
    else:
        flat = np.concatenate([ids[i, : int(lens[i])] for i in range(ids.shape[0])])
    _, cnt = np.unique(flat, return_counts=True)
    cnt = np.sort(cnt)[::-1]
    top = max(1, int(math.ceil(0.2 * cnt.shape[0])))
    return float(cnt[:top].sum() / cnt.sum())
