"""Host logic of the multi-GPU slab sharding (paper_1903_10367_b200.sharding) on CPU.

The sharded schedule runs over CPU numpy shards (tests/sharded_numpy.py) --
in one process (LocalTransport) and as two gloo ranks (DistTransport, the
same torch.distributed calls the NCCL path makes) -- and must reproduce the
serial 3D oracle: every owned plane of u bit for bit, residual history to
1e-13 (the sum of squares is reduced per rank, then across ranks).
"""

import os
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mg3d
from paper_1903_10367_b200 import sharding, workloads
from sharded_numpy import NumpyShard


def test_plan_covers_nests_and_balances():
    for world in (1, 2, 3, 4, 8):
        for depth in (3, 4, 5, 6):
            try:
                pl = sharding.plan(depth, world)
            except ValueError:
                assert 3**depth - 1 < 3 * world
                continue
            for l in range(pl.ls, depth + 1):
                N = 3**l + 1
                rs = pl.own[l]
                assert rs[0][0] == 0 and rs[-1][1] == N
                for r in range(world - 1):
                    assert rs[r][1] == rs[r + 1][0]
                for r in range(world):
                    lo, hi = pl.interior(l, r)
                    assert hi - lo >= 3
                    if l > pl.ls:  # a fine plane 3A + r is owned with coarse plane A
                        clo, chi = pl.own[l - 1][r]
                        assert rs[r][0] == 3 * clo
                        assert rs[r][1] == min(3 * chi, N)
    assert sharding.plan(6, 8).ls == 4 and sharding.plan(6, 8).balanced(4)
    assert sharding.plan(6, 2).ls == 2


def oracle_hist(wl, n, variant=None, flavor=None):
    t = mg3d.Tree(wl.tree.depth, wl.tree.lmin)
    t.eps[wl.tree.depth] = wl.tree.eps[wl.tree.depth].copy()
    e = mg3d.Engine(t, mg3d.Config(variant=variant or wl.variant, flavor=flavor or wl.flavor))
    e.rhs.update({l: b.copy() for l, b in wl.rhs.items()})
    return t, [e.advance() for _ in range(n)]


def check_shard(t, hist, shard, pl, rank, ohist):
    np.testing.assert_allclose([s.l2h for s in hist], [s.l2h for s in ohist], rtol=1e-13)
    assert [s.linf for s in hist] == [s.linf for s in ohist]
    for l in range(pl.ls, t.depth + 1):
        lo, hi = pl.rng(l, rank)
        assert np.array_equal(shard.t.u[l][lo:hi], t.u[l][lo:hi]), f"level {l} rank {rank}"
    for l in range(t.lmin, pl.ls):  # replicated levels: whole array
        assert np.array_equal(shard.t.u[l], t.u[l]), f"replicated level {l}"


CASES = [("config3", 3, "adafac-jac", "geometric"), ("config5", 3, "adafac-jac", "boxmg"),
         ("config5", 3, "additive", "boxmg"), ("config3", 3, "afacc", "geometric"),
         ("config3", 4, "adafac-jac", "geometric")]


@pytest.mark.parametrize("fuse", [False, True])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,levels,variant,flavor", CASES)
def test_local_sharded_equals_oracle(world, name, levels, variant, flavor, fuse):
    mk = workloads.config3 if name == "config3" else workloads.config5
    wl = mk(levels=levels)
    try:
        pl = sharding.plan(levels, world)
    except ValueError:
        pytest.skip("too shallow for this world size")
    shards = [NumpyShard(wl, pl, r, variant, flavor, fuse=fuse) for r in range(world)]
    eng = sharding.ShardedEngine3(shards, sharding.LocalTransport(pl), variant)
    n = 4
    hist = eng.run(n)
    t, oh = oracle_hist(wl, n, variant, flavor)
    for r, s in enumerate(shards):
        check_shard(t, s.history(n), s, pl, r, oh)
    assert hist == shards[0].history(n)


def _gloo_worker(rank, world, port, outdir, name, levels, variant, flavor, fuse=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mk = workloads.config3 if name == "config3" else workloads.config5
        wl = mk(levels=levels)
        pl = sharding.plan(levels, world)
        shard = NumpyShard(wl, pl, rank, variant, flavor, fuse=fuse)
        eng = sharding.ShardedEngine3([shard], sharding.DistTransport(pl, rank), variant)
        hist = eng.run(3)
        np.savez(os.path.join(outdir, f"r{rank}.npz"),
                 l2h=[s.l2h for s in hist], linf=[s.linf for s in hist],
                 **{f"u{l}": shard.t.u[l] for l in range(wl.tree.lmin, levels + 1)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,variant,flavor,fuse", [("config3", "adafac-jac", "geometric", False),
                                                      ("config5", "adafac-jac", "boxmg", False),
                                                      ("config5", "adafac-jac", "boxmg", True)])
def test_gloo_two_ranks_equal_oracle(name, variant, flavor, fuse):
    world, levels = 2, 3
    port = 29500 + (os.getpid() % 1000) + (7 if fuse else 0)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(world, port, d, name, levels, variant, flavor, fuse), nprocs=world,
                 join=True)
        mk = workloads.config3 if name == "config3" else workloads.config5
        wl = mk(levels=levels)
        pl = sharding.plan(levels, world)
        t, oh = oracle_hist(wl, 3, variant, flavor)
        for r in range(world):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            np.testing.assert_allclose(z["l2h"], [s.l2h for s in oh], rtol=1e-13)
            for l in range(pl.ls, levels + 1):
                lo, hi = pl.rng(l, r)
                assert np.array_equal(z[f"u{l}"][lo:hi], t.u[l][lo:hi])
