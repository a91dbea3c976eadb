"""Multi-GPU slab sharding of the 3D cycle.

The finest levels ``ls..ltop`` are cut into slabs of vertex planes along
axis 0 (i, the slowest index, so a slab and every halo plane are contiguous
in memory); level ``ls`` is chosen so every rank owns the same number (>= 3)
of interior planes there, and the cut is refined by 3 per level above it, so
a fine plane ``3A + r`` is owned by the owner of coarse plane ``A``.  Levels
below ``ls`` (a few MB) are replicated and computed redundantly on every
rank.  One process per GPU; the reference is serial, so this
module has no reference counterpart.

Per cycle, phase by phase (``tmg3_phase`` / ``tmg3_phase_range``), with the data exchanges
between phases.  A phase whose result a neighbour needs is split: the planes the neighbour needs
are computed first and their exchange is started, the rest of the owned planes is computed while
the exchange is in flight (NCCL runs on its own stream; the engine's stream waits for it only
where the received planes are read).

==========================  ==================================================
phase                       exchange
==========================  ==================================================
(cycle start)               u_l, every sharded l, ONE batch: plane a-1 from
                            r-1 and b from r+1 -- in flight during the first
                            half of DOWN(ltop)'s inner planes
DOWN(l), l = ltop..ls       rho_l: planes a-2, a-1 from rank r-1, b from r+1
  edge planes first         (a-3 .. a-1 and b when l is fused, below) -- in
  then the inner planes     flight during the inner planes
SMR(l) (adaFACx, l > ls,    -- (the smoothing of l runs fused with the
tmg3_fused; else SMOOTH)    restriction into the owned planes of l-1: sm
                            never leaves the chip, DOWN(l-1) reads b_R, b_T)
SMOOTH(l) (adaFACx)         sm_l: planes a-2, a-1 from rank r-1
(l == ls)                   all-gather rho_ls, sm_ls (the replicated level
                            ls-1 restricts from them)
REDUCE                      all-reduce (sum of squares, max) of the residual
REPL (levels lmin..ls-1)    --
UP(l), l = ls..ltop         carry_l plane a to rank r-1 (read by its UP(l+1)):
  plane a first, then the   in flight during the rest of UP(l)
  rest
(after all UP)              all-gather u_ls, then INJECT into the replicated
                            levels (the u halos move at the next cycle's start;
                            ``sync_halos`` moves them on demand)
==========================  ==================================================

The exchanges are P2P send/recv and collectives on zero-copy torch views of
the engine's device buffers, issued on the engine's own CUDA stream, so
kernels and transfers are ordered without host synchronisation.  The same
schedule drives CPU numpy shards over ``gloo`` in the tests
(tests/test_sharding.py), which is how the host logic is checked without
several GPUs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi

__all__ = ["choose_ls", "plan", "Plan", "DistTransport", "LocalTransport", "GpuShard",
           "ShardedEngine3"]


def choose_ls(depth: int, world: int, lmin: int = 1) -> int:
    """Coarsest level with >= 3 interior planes per rank and an even split (else the
    coarsest with >= 3 per rank)."""
    cands = [l for l in range(lmin + 1, depth + 1) if 3**l - 1 >= 3 * world]
    if not cands:
        raise ValueError(f"depth {depth} is too shallow to shard over {world} ranks")
    for l in cands:
        if (3**l - 1) % world == 0:
            return l
    return cands[0]


@dataclass
class Plan:
    depth: int
    world: int
    ls: int
    own: dict  # level -> list of (lo, hi) vertex-plane ranges, one per rank

    def rng(self, level: int, rank: int) -> tuple[int, int]:
        return self.own[level][rank]

    def interior(self, level: int, rank: int) -> tuple[int, int]:
        lo, hi = self.own[level][rank]
        N = 3**level + 1
        return max(lo, 1), min(hi, N - 1)

    def balanced(self, level: int) -> bool:
        sizes = {self.interior(level, r)[1] - self.interior(level, r)[0] for r in range(self.world)}
        return len(sizes) == 1


def plan(depth: int, world: int, lmin: int = 1, ls: int | None = None) -> Plan:
    ls = choose_ls(depth, world, lmin) if ls is None else ls
    n = 3**ls - 1
    q, rem = divmod(n, world)
    sizes = [q + (1 if r < rem else 0) for r in range(world)]
    if min(sizes) < 3:
        raise ValueError("every rank must own at least 3 interior planes at the shard level")
    cuts = [0]
    acc = 1
    for r in range(world - 1):
        acc += sizes[r]
        cuts.append(acc)
    cuts.append(3**ls + 1)
    own = {}
    for l in range(ls, depth + 1):
        f = 3 ** (l - ls)
        N = 3**l + 1
        own[l] = [(cuts[r] * f, min(cuts[r + 1] * f, N)) for r in range(world)]
    return Plan(depth, world, ls, own)


# ---------------------------------------------------------------------------
# transports: how halo planes, gathers and reductions move between shards


class DistTransport:
    """torch.distributed (NCCL on GPUs, gloo on CPU) for one rank per process."""

    def __init__(self, pl: Plan, rank: int):
        import torch.distributed as dist
        self.dist, self.pl, self.rank = dist, pl, rank

    def halo_begin(self, items):
        """items: (views, level, w_dn, w_up) per field; views[0] is this rank's (N,N,N) view.
        Start ONE batch that receives w_dn planes below the owned range from rank-1 and w_up
        above it from rank+1 (and sends the matching owned planes), for every item.  The batch is
        ordered after the work already enqueued on the current stream; returns the pending
        requests for halo_end."""
        d, r, R = self.dist, self.rank, self.pl.world
        ops = []
        for views, level, w_dn, w_up in items:
            v = views[0]
            a, b = self.pl.rng(level, r)
            if r > 0:
                if w_up:
                    ops.append(d.P2POp(d.isend, v[a:a + w_up], r - 1))
                if w_dn:
                    ops.append(d.P2POp(d.irecv, v[a - w_dn:a], r - 1))
            if r < R - 1:
                if w_dn:
                    ops.append(d.P2POp(d.isend, v[b - w_dn:b], r + 1))
                if w_up:
                    ops.append(d.P2POp(d.irecv, v[b:b + w_up], r + 1))
        return d.batch_isend_irecv(ops) if ops else []

    def halo_end(self, pending) -> None:
        """The current stream (the host, on CPU) waits for the exchange."""
        for req in pending:
            req.wait()

    def halo(self, views, level: int, w_dn: int, w_up: int) -> None:
        self.halo_end(self.halo_begin([(views, level, w_dn, w_up)]))

    def gather(self, views, level: int) -> None:
        """Fill every interior plane of views[0] from its owner."""
        import torch
        d, pl, r = self.dist, self.pl, self.rank
        v = views[0]
        N = v.shape[0]
        lo, hi = pl.interior(level, r)
        if pl.balanced(level):
            d.all_gather_into_tensor(v[1:N - 1], v[lo:hi].clone())
            return
        m = max(pl.interior(level, q)[1] - pl.interior(level, q)[0] for q in range(pl.world))
        send = torch.zeros((m,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)
        send[:hi - lo] = v[lo:hi]
        out = torch.empty((pl.world * m,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)
        d.all_gather_into_tensor(out, send)
        for q in range(pl.world):
            ql, qh = pl.interior(level, q)
            v[ql:qh] = out[q * m:q * m + (qh - ql)]

    def reduce(self, parts) -> None:
        d = self.dist
        p = parts[0]
        d.all_reduce(p[0:1], op=d.ReduceOp.SUM)
        d.all_reduce(p[1:2], op=d.ReduceOp.MAX)


class LocalTransport:
    """All shards in one process (tests on one GPU or on CPU): views is the list of
    every shard's view, in rank order; copies are plain tensor / array copies."""

    def __init__(self, pl: Plan, sync=None):
        self.pl, self.sync = pl, sync

    def _s(self):
        if self.sync:
            self.sync()

    def halo_begin(self, items):
        """Snapshot the planes to be sent NOW (a plane computed after this call does not travel);
        halo_end delivers them (a halo plane read before halo_end is stale) -- the semantics of
        the asynchronous exchange, so the tests see a wrong split."""
        self._s()
        R = self.pl.world
        out = []
        for views, level, w_dn, w_up in items:
            for r in range(R):
                a, b = self.pl.rng(level, r)
                if r > 0 and w_dn:
                    out.append((views[r], a - w_dn, a, views[r - 1][a - w_dn:a].clone()))
                if r < R - 1 and w_up:
                    out.append((views[r], b, b + w_up, views[r + 1][b:b + w_up].clone()))
        self._s()
        return out

    def halo_end(self, pending) -> None:
        self._s()
        for dst, lo, hi, data in pending:
            dst[lo:hi] = data
        self._s()

    def halo(self, views, level: int, w_dn: int, w_up: int) -> None:
        self.halo_end(self.halo_begin([(views, level, w_dn, w_up)]))

    def gather(self, views, level: int) -> None:
        self._s()
        for r in range(self.pl.world):
            for q in range(self.pl.world):
                if q != r:
                    lo, hi = self.pl.interior(level, q)
                    views[r][lo:hi] = views[q][lo:hi]
        self._s()

    def reduce(self, parts) -> None:
        self._s()
        s = sum(float(p[0]) for p in parts)
        m = max(float(p[1]) for p in parts)
        for p in parts:
            p[0] = s
            p[1] = m
        self._s()


# ---------------------------------------------------------------------------
# the GPU shard: one GpuEngine (3D) restricted to its slab


class _CAI:
    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class GpuShard:
    """Phase-level access to a sharded 3D GpuEngine."""

    def __init__(self, eng, pl: Plan, rank: int):
        import ctypes as C
        import torch
        self.eng, self.pl, self.rank = eng, pl, rank
        L = _abi.lib()
        top = eng.ltop
        lo = (C.c_int32 * (top + 1))()
        hi = (C.c_int32 * (top + 1))()
        for l in range(pl.ls, top + 1):
            lo[l], hi[l] = pl.rng(l, rank)
        _abi.check(L.tmg3_shard(eng._h, pl.ls, lo, hi))
        s = C.c_uint64()
        _abi.check(L.tmg3_stream(eng._h, C.byref(s)))
        self.stream = torch.cuda.ExternalStream(s.value, device=torch.device("cuda", eng.device))
        self._views = {}

    def view(self, field: int, level: int):
        # the finest level's u is double buffered: its current buffer alternates every cycle
        key = (field, level, self.state()[1] if field == _abi.F_U and level == self.eng.ltop else 0)
        if key not in self._views:
            import ctypes as C
            import torch
            p, n = C.c_uint64(), C.c_int64()
            _abi.check(_abi.lib().tmg3_field(self.eng._h, field, level, C.byref(p), C.byref(n)))
            if field == _abi.F_PART:
                shape = (2,)
            else:
                N = 3**level + 1
                shape = (N, N, N)
            self._views[key] = torch.as_tensor(_CAI(p.value, shape), device=f"cuda:{self.eng.device}")
        return self._views[key]

    def phase(self, ph: int, level: int = 0, rng=None, first: bool = True, last: bool = True) -> None:
        """One phase; ``rng = (lo, hi)`` restricts DOWN / UP to the owned planes inside it
        (``first`` / ``last``: the first / last part of this phase in the cycle)."""
        if rng is None:
            _abi.check(_abi.lib().tmg3_phase(self.eng._h, ph, level))
        else:
            _abi.check(_abi.lib().tmg3_phase_range(self.eng._h, ph, level, int(rng[0]), int(rng[1]),
                                                   1 if first else 0, 1 if last else 0))

    def state(self, new=None):
        """(cycles enqueued, parity of the finest level's double buffer); ``new`` sets it."""
        import ctypes as C
        c, p = C.c_int64(), C.c_int32()
        if new is not None:
            c.value, p.value = new
        _abi.check(_abi.lib().tmg3_cycle_state(self.eng._h, C.byref(c), C.byref(p), 0 if new is None else 1))
        return c.value, p.value

    def fused(self, level: int) -> bool:
        """Whether the engine runs level's smoothing fused with the restriction (PH_SMR)."""
        import ctypes as C
        v = C.c_int32()
        _abi.check(_abi.lib().tmg3_fused(self.eng._h, level, C.byref(v)))
        return bool(v.value)

    def close(self) -> None:
        """Drop the zero-copy views (call before the engine is closed)."""
        self._views.clear()

    def history(self, n: int):
        import ctypes as C
        out = (_abi.Stats * max(n, 1))()
        _abi.check(_abi.lib().tmg3_history(self.eng._h, n, C.cast(out, C.c_void_p)))
        return [self.eng._stats(out[k]) for k in range(n)]


class ShardedEngine3:
    """The sharded cycle (schedule above) over a list of local shards and a transport.

    ``shards`` holds this process's shard(s): one with DistTransport (one rank
    per process), all of them with LocalTransport.
    """

    def __init__(self, shards, transport, variant: str, lmin: int = 1, split: bool | None = None):
        self.shards, self.tr = shards, transport
        self.pl = shards[0].pl
        self.jac = variant == "adafac-jac"
        self.lmin = lmin
        # split the phases a neighbour waits for (edge planes, exchange, inner planes)
        self.split = self.pl.world > 1 if split is None else split
        self._fz = {}
        self._graphs = None

    def _views(self, field, level):
        return [s.view(field, level) for s in self.shards]

    def _fused(self, level) -> bool:
        if level not in self._fz:
            f = {bool(getattr(s, "fused", lambda _l: False)(level)) for s in self.shards}
            if len(f) != 1:
                raise RuntimeError(f"shards disagree on the fused smoothing of level {level}")
            self._fz[level] = f.pop()
        return self._fz[level]

    # -- split phases ---------------------------------------------------------------------
    def _ranks(self):
        return [s.rank for s in self.shards]

    def _phase_parts(self, ph, level, parts, first, last):
        """parts(rank) -> list of (lo, hi) plane ranges; one ranged phase call per range."""
        for s in self.shards:
            rs = [r for r in parts(s.rank) if r[1] > r[0]]
            for k, r in enumerate(rs):
                s.phase(ph, level, rng=r, first=first and k == 0, last=last and k == len(rs) - 1)

    def _can_split(self, level, w_dn, w_up) -> bool:
        if not self.split:
            return False
        return all(self.pl.interior(level, r)[1] - self.pl.interior(level, r)[0] >= w_dn + w_up + 2
                   for r in range(self.pl.world))

    def _down(self, l, w_dn, w_up, pend_u=None):
        """DOWN(l) followed by the rho halo (w_dn planes below, w_up above).  Split: the planes a
        neighbour receives -- the first w_up and the last w_dn owned planes -- first, then the
        exchange in flight during the inner planes.  ``pend_u`` (finest level): the u halos started
        at the top of the cycle; only the first and the last owned plane read them, so half of the
        inner planes run before they are waited for."""
        pl, tr = self.pl, self.tr
        rho = self._views(_abi.F_RHO, l)
        if not self._can_split(l, w_dn, w_up):
            if pend_u is not None:
                tr.halo_end(pend_u)
            for s in self.shards:
                s.phase(_abi.PH_DOWN, l)
            tr.halo(rho, l, w_dn, w_up)
            return
        first = True
        mid = {}
        for r in range(pl.world):
            a, b = pl.interior(l, r)
            mid[r] = a + w_up + (b - w_dn - a - w_up) // 2 if pend_u is not None else a + w_up
        if pend_u is not None:
            self._phase_parts(_abi.PH_DOWN, l, lambda r: [(pl.interior(l, r)[0] + w_up, mid[r])], True, False)
            first = False
            tr.halo_end(pend_u)
        self._phase_parts(_abi.PH_DOWN, l, lambda r: [(pl.interior(l, r)[0], pl.interior(l, r)[0] + w_up),
                                                       (pl.interior(l, r)[1] - w_dn, pl.interior(l, r)[1])],
                          first, False)
        pend = tr.halo_begin([(rho, l, w_dn, w_up)])
        self._phase_parts(_abi.PH_DOWN, l, lambda r: [(mid[r], pl.interior(l, r)[1] - w_dn)], False, True)
        tr.halo_end(pend)

    def cycle(self) -> None:
        pl, tr = self.pl, self.tr
        ls, top = pl.ls, pl.depth
        # the iterate's halo planes (of the previous cycle's update), every sharded level in one batch
        pend_u = tr.halo_begin([(self._views(_abi.F_U, l), l, 1, 1) for l in range(ls, top + 1)])
        for l in range(top, ls - 1, -1):
            pu = pend_u if l == top else None
            if self.jac and l > ls and self._fused(l):
                # smoothing fused with the restriction into l - 1 (sm stays on chip): rho needs
                # the 3 planes below (sm of the 2 below) and 1 above, no sm halo
                self._down(l, 3, 1, pu)
                for s in self.shards:
                    s.phase(_abi.PH_SMR, l)
                continue
            self._down(l, 2, 1, pu)
            if self.jac:
                for s in self.shards:
                    s.phase(_abi.PH_SMOOTH, l)
                if l > ls:
                    tr.halo(self._views(_abi.F_SM, l), l, 2, 0)
            if l == ls:
                tr.gather(self._views(_abi.F_RHO, l), l)
                if self.jac:
                    tr.gather(self._views(_abi.F_SM, l), l)
        for s in self.shards:
            s.phase(_abi.PH_REDUCE)
        tr.reduce(self._views(_abi.F_PART, 0))
        for s in self.shards:
            s.phase(_abi.PH_REPL)
        pend = None
        for l in range(ls, top + 1):
            if pend is not None:
                tr.halo_end(pend)  # carry_{l-1}: plane b from rank r+1
                pend = None
            if l < top and self._can_split(l, 0, 1):
                # the first owned plane of carry_l goes to rank r-1 while the rest of UP(l) runs
                self._phase_parts(_abi.PH_UP, l, lambda r: [(pl.interior(l, r)[0], pl.interior(l, r)[0] + 1)],
                                  True, False)
                pend = tr.halo_begin([(self._views(_abi.F_CARRY, l), l, 0, 1)])
                self._phase_parts(_abi.PH_UP, l, lambda r: [(pl.interior(l, r)[0] + 1, pl.interior(l, r)[1])],
                                  False, True)
            else:
                for s in self.shards:
                    s.phase(_abi.PH_UP, l)
                if l < top:
                    pend = tr.halo_begin([(self._views(_abi.F_CARRY, l), l, 0, 1)])
        tr.gather(self._views(_abi.F_U, ls), ls)
        for s in self.shards:
            s.phase(_abi.PH_INJECT)

    def sync_halos(self) -> None:
        """Move the iterate's halo planes now (the cycle moves them at its start)."""
        pl = self.pl
        self.tr.halo_end(self.tr.halo_begin([(self._views(_abi.F_U, l), l, 1, 1)
                                             for l in range(pl.ls, pl.depth + 1)]))

    def run(self, n: int):
        for _ in range(n):
            self.cycle()
        self.sync_halos()  # leave the iterate's halo planes current
        return self.shards[0].history(n)

    # -- the cycle as CUDA graphs (one process per GPU) -----------------------------------
    def capture(self) -> bool:
        """Capture the cycle -- every phase kernel and every NCCL exchange between them, all on
        the engine's stream -- into two CUDA graphs, one per parity of the finest level's double
        buffer, so a cycle costs one graph launch instead of ~40 host enqueues.  Returns False
        (and stays on the eager path) if the capture fails."""
        import torch
        if len(self.shards) != 1:
            raise RuntimeError("graph capture is for one shard per process")
        sh = self.shards[0]
        before = sh.state()
        graphs, pool = [], None
        try:
            for _ in range(2):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, pool=pool, stream=sh.stream, capture_error_mode="thread_local"):
                    self.cycle()
                pool = g.pool()
                graphs.append(g)
        except Exception as exc:  # stay on the eager path
            import sys
            print(f"sharded cycle: CUDA graph capture failed ({exc!r}); running eagerly", file=sys.stderr)
            sh.state(before)
            self._graphs = None
            return False
        sh.state(before)  # the captured cycles did not run
        self._graphs, self._next = graphs, 0
        return True

    def replay(self) -> None:
        """One cycle from the captured graphs (launch on the shard's stream)."""
        self._graphs[self._next].replay()
        c, p = self.shards[0].state()
        self.shards[0].state((c + 1, p ^ 1))
        self._next ^= 1


def owned_u(pl: Plan, level: int, rank: int, u: np.ndarray) -> np.ndarray:
    """The planes of u a rank owns (for assembling a global iterate in tests)."""
    lo, hi = pl.rng(level, rank)
    return u[lo:hi]
