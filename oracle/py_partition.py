"""Python restatement of the reference's multilevel k-way partitioner
(/root/reference/pkg/src/splatsched/partition.py:104-434).

TEST INFRASTRUCTURE ONLY (oracle/): the product runs the native C++ port
(paper_2512_20017_b200/csrc/host/partition.cpp); tests check that port
against this restatement on random graphs and against the reference's own
golden labels (tests/golden)."""

from __future__ import annotations

import numpy as np

from paper_2512_20017_b200.sharding import COARSEN_FACTOR, WeightedGraph


class Multilevel:
    """One run of the multilevel k-way scheme with its own PCG64 stream."""

    def __init__(self, parts: int, eps: float, rng: np.random.Generator):
        self.k, self.eps, self.rng = parts, eps, rng

    # -- coarsening -------------------------------------------------------
    def contract(self, g: WeightedGraph, cap: float):
        mate = np.full(g.n, -1, dtype=np.int64)
        for v in range(g.n):
            if mate[v] != -1:
                continue
            nb, ws = g.nbrs(v)
            ok = (mate[nb] == -1) & (nb != v) & ~(g.bal[v] + g.bal[nb] > cap)
            if not ok.any():
                continue
            heavy = ws[ok].max()
            pool = nb[ok & (ws == heavy)]
            u = int(pool[self.rng.integers(len(pool))]) if len(pool) > 1 else int(pool[0])
            mate[v], mate[u] = u, v
        if (mate == -1).all():
            return None
        cid = np.full(g.n, -1, dtype=np.int64)
        nxt = 0
        for v in range(g.n):
            if cid[v] == -1:
                cid[v] = nxt
                if mate[v] != -1:
                    cid[mate[v]] = nxt
                nxt += 1
        cbal = np.zeros(nxt)
        np.add.at(cbal, cid, g.bal)
        a, b = cid[g.eu], cid[g.ev]
        keep = a != b
        a, b, w = a[keep], b[keep], g.ew[keep]
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        key = lo * nxt + hi
        o = np.argsort(key, kind="stable")
        key, lo, hi, w = key[o], lo[o], hi[o], w[o]
        _, first = np.unique(key, return_index=True)
        merged = np.add.reduceat(w, first) if len(w) else w
        return WeightedGraph(nxt, cbal, lo[first], hi[first], merged), cid

    # -- initial partition ---------------------------------------------------
    def grow(self, g: WeightedGraph):
        k = self.k
        lab = np.full(g.n, -1, dtype=np.int64)
        left = g.n
        goal = g.bal.sum() / k
        link = np.zeros(g.n)
        for part in range(k - 1):
            if left <= k - part - 1:
                break
            free = np.flatnonzero(lab == -1)
            cur = int(free[self.rng.integers(len(free))])
            link[:] = 0.0
            mass = 0.0
            while True:
                lab[cur] = part
                left -= 1
                mass += g.bal[cur]
                nb, ws = g.nbrs(cur)
                open_ = lab[nb] == -1
                link[nb[open_]] += ws[open_]
                if mass >= goal or left <= k - part - 1:
                    break
                free = np.flatnonzero(lab == -1)
                lf = link[free]
                if lf.max() > 0:
                    cur = int(free[int(np.argmax(lf))])
                else:
                    cur = int(free[self.rng.integers(len(free))])
        lab[lab == -1] = k - 1
        return lab

    # -- refinement ------------------------------------------------------------
    @staticmethod
    def _affinity(g: WeightedGraph, lab, k):
        aff = np.zeros((g.n, k))
        np.add.at(aff, (g.eu, lab[g.ev]), g.ew)
        np.add.at(aff, (g.ev, lab[g.eu]), g.ew)
        return aff

    @staticmethod
    def _move(g: WeightedGraph, aff, lab, v, dst):
        src = lab[v]
        nb, ws = g.nbrs(v)
        np.add.at(aff, (nb, src), -ws)
        np.add.at(aff, (nb, dst), ws)
        lab[v] = dst

    def _force_balance(self, g, lab, cap, aff, pw):
        k = self.k
        budget = 10 * g.n + 10
        while budget > 0:
            over = np.flatnonzero(pw > cap)
            if len(over) == 0:
                return True
            budget -= 1
            heavy = int(over[np.argmax(pw[over])])
            cand = np.flatnonzero((lab == heavy) & (g.bal > 0))
            if len(cand) == 0:
                return False
            room = cap - (pw[None, :] + g.bal[cand][:, None])
            tgt = np.broadcast_to(np.arange(k), room.shape)
            okm = (tgt != heavy) & ~(room < 0)
            if not okm.any():
                return False
            vv = np.broadcast_to(cand[:, None], room.shape)[okm]
            tt = tgt[okm]
            ng = -(aff[vv, tt] - aff[vv, heavy])
            pick = np.lexsort((tt, vv, pw[tt], ng))[0]
            v, t = int(vv[pick]), int(tt[pick])
            pw[heavy] -= g.bal[v]
            pw[t] += g.bal[v]
            self._move(g, aff, lab, v, t)
        return bool((g.part_weights(lab, k) <= cap).all())

    def refine(self, g: WeightedGraph, lab, cap):
        k, n = self.k, g.n
        limit = 100 * n + 100
        aff = self._affinity(g, lab, k)
        pw = g.part_weights(lab, k)
        self._force_balance(g, lab, cap, aff, pw)
        rows = np.arange(n)
        for _ in range(limit):
            gain = aff - aff[rows, lab][:, None]
            gain = np.where((pw[None, :] + g.bal[:, None]) <= cap, gain, -np.inf)
            gain[rows, lab] = -np.inf
            top = gain.max()
            if top < 0:
                break
            if top > 0:
                v, t = divmod(int(np.argmax(gain)), k)
            else:
                v = t = -1
                best = 0.0
                for cv, ct in np.argwhere(gain == 0.0):
                    w = g.bal[cv]
                    if w == 0:
                        continue
                    delta = 2.0 * w * (pw[ct] - pw[lab[cv]] + w)
                    if delta < best - 1e-12:
                        best, v, t = delta, int(cv), int(ct)
                if v == -1:
                    break
            pw[lab[v]] -= g.bal[v]
            pw[t] += g.bal[v]
            self._move(g, aff, lab, v, t)
        return lab

    def run(self, g: WeightedGraph):
        cap = (1.0 + self.eps) * g.bal.sum() / self.k
        stack, maps = [g], []
        cur = g
        while cur.n > COARSEN_FACTOR * self.k:
            res = self.contract(cur, cap)
            if res is None:
                break
            cur, cid = res
            stack.append(cur)
            maps.append(cid)
            if stack[-2].n - cur.n < max(1, stack[-2].n // 20):
                break
        lab = self.refine(stack[-1], self.grow(stack[-1]), cap)
        for level in range(len(maps) - 1, -1, -1):
            lab = self.refine(stack[level], lab[maps[level]], cap)
        return lab
