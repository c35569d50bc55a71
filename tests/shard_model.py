"""Numpy model of one rank of the A-row-sharded phase step (test
infrastructure only: it lets the CPU suite drive the same
paper_2203_03732_b200.sharded.run_phases protocol, including the gloo
world_size-2 exchange, and check it against the oracle).

It mirrors csrc/shard_kernels.cu step by step (top / compact / scan / DA with
parking), with chains processed one at a time: deferred acceptance has one
outcome whatever the interleaving, so the sequential model and the parallel
kernels must agree with the reference's sequential greedy
(assignment.cpp:161-171) — which is what the tests check.
"""
from __future__ import annotations

import numpy as np

TAG_SHIFT = np.uint64(32)
ALL_ONES = np.uint64(0xFFFFFFFFFFFFFFFF)


class NumpyRank:
    def __init__(self, align: int = 512):
        self.align = align

    # kT: (ib, ia) int matrix, internal orientation (ia >= ib)
    def prepare(self, kT: np.ndarray, eps: float, n_shards: int, shard: int, K: int = 16):
        ib, ia = kT.shape
        bounds = [(ia * g // n_shards) // self.align * self.align for g in range(n_shards)]
        self.bounds = np.array(bounds + [ia], np.int64)
        self.lo, self.hi = int(self.bounds[shard]), int(self.bounds[shard + 1])
        self.slab = np.ascontiguousarray(kT[:, self.lo:self.hi]).astype(np.int64)
        self.ia, self.ib, self.eps = ia, ib, eps
        self.n_shards, self.shard, self.K = n_shards, shard, K
        self.cap = ib
        self.thresh = int(np.floor(eps * min(ia, ib)))
        self.phase_cap = int(np.ceil((1.0 + 2.0 * eps) / (eps * eps))) + 8
        return self.bounds

    def begin(self):
        self.t = np.zeros(self.ia, np.int64)
        self.yb = np.ones(self.ib, np.int64)
        self.ma = np.full(self.ia, -1, np.int64)
        self.mb = np.full(self.ib, -1, np.int64)
        self.holder = np.full(self.ia, ALL_ONES, np.uint64)
        self.cnt = [self.ib, 0]
        self.mp = [[], []]
        self.phase = 0
        self.free_counts = []
        self.sum_ni = 0
        self.done = False
        self.parked = []

    def top(self):
        p = self.phase
        par = p & 1
        if p > 0:
            for a, old_b in self.mp[par]:
                b = int(self.holder[a] & np.uint64(0xFFFFFFFF))
                if old_b >= 0:
                    self.mb[old_b] = -1
                self.ma[a] = b
                self.mb[b] = a
                self.t[a] += 1
        n = self.cnt[par]
        if n <= self.thresh:
            self.done = True
            self.full_match = n == 0
            return n, True
        if p + 1 > self.phase_cap:
            raise RuntimeError("phase cap exceeded")
        self.free_counts.append(n)
        self.sum_ni += n
        nx = par ^ 1
        self.cnt[nx] = 0
        self.mp[nx] = []
        self.list = np.flatnonzero(self.mb == -1)
        assert len(self.list) == n, (len(self.list), n)
        self.pos = {int(b): i for i, b in enumerate(self.list)}
        return n, False

    def scan(self, cand, meta, cap, refill):
        K, g = self.K, self.shard
        reqs = self.parked if refill else [(i, int(b), 0) for i, b in enumerate(self.list)]
        for i, b, start in reqs:
            target = self.yb[b] - 1
            row = self.slab[b] + self.t[self.lo:self.hi]
            ls = max(start, self.lo) - self.lo
            hits = np.flatnonzero(row[ls:] == target) + ls + self.lo if start < self.hi else []
            o = (g * cap + i) * K
            cnt = min(len(hits), K)
            cand[o:o + cnt] = hits[:cnt]
            cov = int(hits[K - 1]) + 1 if len(hits) >= K else self.hi
            meta[2 * (g * cap + i)] = cnt
            meta[2 * (g * cap + i) + 1] = cov

    def da(self, cand, meta, cap, resume):
        phase = self.phase + 1
        tag = np.uint64(~np.uint32(phase) & np.uint32(0xFFFFFFFF))
        par = phase & 1
        chains = self.parked if resume else [(i, int(b), 0) for i, b in enumerate(self.list)]
        parked = []
        for i, b, start in chains:
            while True:
                a, restart = -1, -1
                for g in range(self.n_shards):
                    ghi = int(self.bounds[g + 1])
                    if start >= ghi:
                        continue
                    c, cov = int(meta[2 * (g * cap + i)]), int(meta[2 * (g * cap + i) + 1])
                    lst = [int(x) for x in cand[(g * cap + i) * self.K:(g * cap + i) * self.K + c]]
                    hit = [x for x in lst if x >= start]
                    if hit:
                        a = hit[0]
                        break
                    if cov < ghi:
                        restart = max(start, cov)
                        break
                if a < 0 and restart >= 0:
                    parked.append((i, b, restart))
                    break
                if a < 0:
                    self.yb[b] += 1
                    self.cnt[par] += 1
                    break
                key = (tag << TAG_SHIFT) | np.uint64(b)
                old = self.holder[a]
                self.holder[a] = min(old, key)
                if old < key:
                    start = a + 1
                    continue
                if (old >> TAG_SHIFT) == tag:
                    b = int(old & np.uint64(0xFFFFFFFF))
                    i = self.pos[b]
                    start = a + 1
                    continue
                partner = int(self.ma[a])
                if partner >= 0:
                    self.cnt[par] += 1
                self.mp[par].append((a, partner))
                break
        self.parked = parked
        if not parked:
            self.phase += 1
        return len(parked)

    def finish(self):
        ma, mb = self.ma.copy(), self.mb.copy()
        fa = np.flatnonzero(ma == -1)
        fb = np.flatnonzero(mb == -1)
        for a, b in zip(fa, fb):
            ma[a], mb[b] = b, a
        return dict(match_of_a=ma, match_of_b=mb, y_a=-self.t, y_b=self.yb.copy(),
                    phases=self.phase, sum_ni=self.sum_ni,
                    free_counts=np.array(self.free_counts, np.int64))
