"""Sharded 3D cycle on the GPU kernels (one B200 available).

Several GpuShards (each a full GpuEngine restricted to its slab with
tmg3_shard) run in ONE process on cuda:0 and exchange planes with
LocalTransport (device copies between their buffers, streams synchronised at
every exchange), so no rank ever waits on another rank's kernel.  The result
must equal the unsharded GPU engine up to round-off (u on every owned plane
within 1e-12 normwise): the unsharded cycle keeps the finest level double
buffered (u + g written by the down sweep), the phase-by-phase sharded cycle
adds g in the up sweep, so the two round differently.  A
world-size-1 NCCL process group exercises DistTransport's collectives on
zero-copy views of the engine buffers on the engine's stream.
"""

import os

import numpy as np
import pytest
import torch

from paper_1903_10367_b200 import GpuEngine, SolverConfig, sharding, workloads

pytestmark = pytest.mark.gpu


def close(got, want, rtol=1e-12, what="u"):
    err = float(np.abs(got - want).max())
    assert err <= rtol * max(float(np.abs(want).max()), 1e-300), f"{what}: {err:.3e}"


def serial(wl, n, variant, **kw):
    eng = GpuEngine(wl.tree, SolverConfig(variant=variant, flavor=wl.flavor, **kw), sync="lazy")
    eng.rhs.update(wl.rhs)
    h = eng.advance_many(n)
    eng.pull()
    return h


def sharded_local(mk, world, n, variant, **kw):
    wl0 = mk()
    pl = sharding.plan(wl0.tree.depth, world)
    shards, wls = [], []
    for r in range(world):
        wl = mk()
        eng = GpuEngine(wl.tree, SolverConfig(variant=variant, flavor=wl.flavor, **kw), sync="lazy")
        eng.rhs.update(wl.rhs)
        eng._flush_rhs()
        shards.append(sharding.GpuShard(eng, pl, r))
        wls.append(wl)
    se = sharding.ShardedEngine3(shards, sharding.LocalTransport(pl, sync=torch.cuda.synchronize), variant)
    h = se.run(n)
    for s in shards:
        s.eng.pull()
    return pl, wls, shards, h


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,variant", [("config5-L4", "adafac-jac"), ("config3-L4", "adafac-jac"),
                                          ("config5-L4", "additive"), ("config3-L4", "afacc"),
                                          ("config5-L5", "adafac-jac")])
def test_gpu_sharded_equals_serial(world, name, variant):
    mk = lambda: workloads.by_name(name)  # noqa: E731
    wl = mk()
    n = 4
    hs = serial(wl, n, variant)
    pl, wls, shards, h = sharded_local(mk, world, n, variant)
    np.testing.assert_allclose([s.l2h for s in h], [s.l2h for s in hs], rtol=1e-12)
    np.testing.assert_allclose([s.linf for s in h], [s.linf for s in hs], rtol=1e-12)
    top = wl.tree.depth
    for r in range(world):
        for l in range(pl.ls, top + 1):
            lo, hi = pl.rng(l, r)
            close(wls[r].tree.u[l][lo:hi], wl.tree.u[l][lo:hi], what=f"rank {r} level {l}")
        for l in range(wl.tree.lmin, pl.ls):
            close(wls[r].tree.u[l], wl.tree.u[l], what=f"rank {r} replicated level {l}")
    if variant == "adafac-jac" and name.startswith("config5"):
        # BoxMG adaFACx: the finest level's smoothing runs fused with the restriction (PH_SMR)
        assert shards[0].fused(top) and not shards[0].fused(pl.ls)


def test_gpu_sharded_throttled_equals_serial():
    """Throttled setup in the sharded schedule: the level upgrade runs at the top DOWN phase."""
    mk = lambda: workloads.by_name("config5-L4")  # noqa: E731
    wl = mk()
    n = 5
    hs = serial(wl, n, "adafac-jac", throttled=True)
    pl, wls, shards, h = sharded_local(mk, 2, n, "adafac-jac", throttled=True)
    np.testing.assert_allclose([s.l2h for s in h], [s.l2h for s in hs], rtol=1e-12)
    for r in range(2):
        lo, hi = pl.rng(wl.tree.depth, r)
        close(wls[r].tree.u[wl.tree.depth][lo:hi], wl.tree.u[wl.tree.depth][lo:hi])


def test_gpu_dist_transport_world1_nccl():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29631")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        wl = workloads.by_name("config5-L4")
        hs = serial(wl, 3, wl.variant)
        wl2 = workloads.by_name("config5-L4")
        pl = sharding.plan(wl2.tree.depth, 1)
        eng = GpuEngine(wl2.tree, SolverConfig(variant=wl2.variant, flavor=wl2.flavor), sync="lazy")
        eng.rhs.update(wl2.rhs)
        eng._flush_rhs()
        sh = sharding.GpuShard(eng, pl, 0)
        se = sharding.ShardedEngine3([sh], sharding.DistTransport(pl, 0), wl2.variant)
        with torch.cuda.stream(sh.stream):
            h = se.run(3)
        eng.pull()
        np.testing.assert_allclose([s.l2h for s in h], [s.l2h for s in hs], rtol=1e-12)
        close(wl2.tree.u[4], wl.tree.u[4])
        sh.close()
        # the split schedule (edge planes, exchange, inner planes: tmg3_phase_range) forced on the
        # single rank, eagerly and replayed from the captured CUDA graphs
        wl3 = workloads.by_name("config5-L4")
        eng3 = GpuEngine(wl3.tree, SolverConfig(variant=wl3.variant, flavor=wl3.flavor), sync="lazy")
        eng3.rhs.update(wl3.rhs)
        eng3._flush_rhs()
        sh3 = sharding.GpuShard(eng3, pl, 0)
        se3 = sharding.ShardedEngine3([sh3], sharding.DistTransport(pl, 0), wl3.variant, split=True)
        with torch.cuda.stream(sh3.stream):
            se3.cycle()
            assert se3.capture()
            se3.replay()
            se3.replay()
        torch.cuda.synchronize()
        h3 = sh3.history(3)
        eng3.pull()
        np.testing.assert_allclose([s.l2h for s in h3], [s.l2h for s in hs], rtol=1e-12)
        close(wl3.tree.u[4], wl.tree.u[4])
        sh3.close()
    finally:
        dist.destroy_process_group()
