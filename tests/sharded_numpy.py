"""CPU shard with the phase API of sharding.GpuShard, computed with the 3D oracle.

Test infrastructure: lets the sharded schedule (paper_1903_10367_b200.sharding)
run on CPU, in one process (LocalTransport) or over gloo (DistTransport), so
the host logic -- which planes move when -- is checked against the serial
oracle without several GPUs.  Every phase evaluates the oracle's primitives on
the full arrays and keeps only the planes the shard owns, so a missing or
misplaced exchange shows up as a wrong iterate.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import mg3d
from paper_1903_10367_b200 import _abi


class NumpyShard:
    def __init__(self, wl, pl, rank, variant=None, flavor=None, fuse=False):
        self.pl, self.rank = pl, rank
        self.fuse = fuse  # emulate tmg3_fused / PH_SMR on the levels above ls
        L = wl.tree.depth
        t = mg3d.Tree(L, wl.tree.lmin)
        t.eps[L] = wl.tree.eps[L].copy()
        self.cfg = mg3d.Config(variant=variant or wl.variant, flavor=flavor or wl.flavor)
        self.e = mg3d.Engine(t, self.cfg)  # operators only
        self.t = t
        self.top, self.l0 = L, wl.tree.lmin
        self.rhs = {l: b.copy() for l, b in wl.rhs.items()}
        z = {l: np.zeros_like(t.u[l]) for l in range(self.l0, L + 1)}
        self.g = {l: z[l].copy() for l in z}
        self.rho = {l: z[l].copy() for l in z}
        self.sm = {l: z[l].copy() for l in z}
        self.carry = {l: z[l].copy() for l in z}
        self.part = np.zeros(2)
        self.hist = []

    # -- views ------------------------------------------------------------------
    def view(self, field, level):
        if field == _abi.F_PART:
            return torch.from_numpy(self.part)
        arr = {_abi.F_U: self.t.u, _abi.F_RHO: self.rho, _abi.F_SM: self.sm,
               _abi.F_CARRY: self.carry, _abi.F_G: self.g}[field][level]
        return torch.from_numpy(arr)

    # -- helpers ----------------------------------------------------------------
    def _own(self, l, rng=None):
        """slice of owned interior planes (i) -- inside rng when given -- and the interior (j, k) box."""
        lo, hi = self.pl.interior(l, self.rank)
        if rng is not None:
            lo, hi = max(lo, rng[0]), min(hi, rng[1])
        return (slice(lo, max(lo, hi)), slice(1, -1), slice(1, -1))

    def _rhs(self, l):
        r = self.rhs.get(l)
        return np.zeros_like(self.t.u[l]) if r is None else r

    def _w(self, l):
        if self.cfg.variant == "additive-exp":
            return self.cfg.omega_hat ** (self.top - l)
        return self.cfg.omega

    def _down(self, l, own, first=True):
        e, cfg = self.e, self.cfg
        op = e.ops[l]
        dof = e.masks[l]["dof"]
        diag = np.where(dof, op.diag(), 1.0)
        au = op.apply(self.t.u[l])
        if l == self.top:
            b = self._rhs(l)
        else:
            src = self.rho[l + 1]
            if cfg.variant == "afacc":
                src = src.copy()
                src[::3, ::3, ::3] = 0.0
            b = e.tr[l].restrict(src)
            b += self._rhs(l)
            b = b + np.where(e.masks[l]["overlapped"], au, 0.0)
        rho = np.where(dof, b - au, 0.0)
        if cfg.variant == "bpx" and l < self.top:
            d = cfg.omega * rho
        else:
            d = self._w(l) * rho / diag
        if cfg.variant == "adafac-jac" and l < self.top:
            bt = e.tr[l].restrict(self.sm[l + 1])
            dt = cfg.damping_scale * (cfg.wt * bt / diag)
            dt[~dof] = 0.0
            d = d - dt
        self.g[l][own] = d[own]
        self.rho[l][own] = rho[own]
        if l == self.top:
            r = rho[own]
            hw = e.hw[l]
            if first:
                self.part[:] = 0.0
            self.part[0] += float(((hw * r) ** 2).sum())
            self.part[1] = max(self.part[1], float(np.abs(r).max()) if r.size else 0.0)

    def _smooth(self, l, own):
        s = mg3d.apply_const(self.rho[l], 1.0)
        s *= self.cfg.omega * 3.0 / 8.0
        self.sm[l][own] = s[own]

    def _up(self, l, own):
        e = self.e
        g = self.g[l]
        if l == self.l0:
            c = g.copy()
        else:
            c = e.tr[l - 1].prolong(self.carry[l - 1]) + g
        self.carry[l][own] = c[own]
        self.t.u[l][own] = self.t.u[l][own] + c[own]

    def _smr(self, l):
        """PH_SMR: sm of the owned planes and of the 2 below them, from this shard's rho alone
        (fresh only with the 3-below / 1-above rho halo), never exchanged; DOWN(l-1) restricts it."""
        s = mg3d.apply_const(self.rho[l], 1.0)
        s *= self.cfg.omega * 3.0 / 8.0
        lo, hi = self.pl.interior(l, self.rank)
        a = max(lo - 2, 1)
        self.sm[l][a:hi, 1:-1, 1:-1] = s[a:hi, 1:-1, 1:-1]

    def fused(self, level):
        return self.fuse and self.cfg.variant == "adafac-jac" and self.pl.ls < level <= self.top

    # -- phases -----------------------------------------------------------------
    def phase(self, ph, level=0, rng=None, first=True, last=True):
        ls, top, l0 = self.pl.ls, self.top, self.l0
        full = (slice(1, -1),) * 3
        if rng is not None:
            assert ph in (_abi.PH_DOWN, _abi.PH_UP)
        if ph == _abi.PH_DOWN:
            self._down(level, self._own(level, rng), first)
        elif ph == _abi.PH_SMOOTH:
            if self.cfg.variant == "adafac-jac" and level > l0:
                self._smooth(level, self._own(level))
        elif ph == _abi.PH_SMR:
            assert self.fused(level), level
            self._smr(level)
        elif ph == _abi.PH_REDUCE:
            pass
        elif ph == _abi.PH_REPL:
            for l in range(ls - 1, l0 - 1, -1):
                self._down(l, full)
                if self.cfg.variant == "adafac-jac" and l > l0:
                    self._smooth(l, full)
            self.hist.append(mg3d.Stats(float(np.sqrt(self.part[0])), float(self.part[1]),
                                        (3**top - 1) ** 3, self.e.count_updates()))
            for l in range(l0, ls):
                self._up(l, full)
        elif ph == _abi.PH_UP:
            own = self._own(level, rng)
            self._up(level, own)
            lo, hi = own[0].start, own[0].stop
            fine = self.t.u[level]
            for lc in range(level - 1, ls - 1, -1):
                # walk-down: fine c-points in owned planes -> coarser sharded levels
                Nc = 3**lc + 1
                step = 3 ** (level - lc)
                W = np.arange(1, Nc - 1)
                Wi = W[(step * W >= lo) & (step * W < hi)]
                if Wi.size:
                    sub = fine[step * Wi][:, step * W][:, :, step * W]
                    self.t.u[lc][Wi[0]:Wi[-1] + 1, 1:-1, 1:-1] = sub
        elif ph == _abi.PH_INJECT:
            for l in range(ls - 1, l0 - 1, -1):
                self.t.u[l][1:-1, 1:-1, 1:-1] = self.t.u[l + 1][::3, ::3, ::3][1:-1, 1:-1, 1:-1]
        else:
            raise ValueError(ph)

    def history(self, n):
        return self.hist[-n:]
