"""CPU (gloo, world_size 2) tests of the multi-rank host logic of the slab decomposition:
slab cuts, per-rank scene generation and the id handshake.  The union of what the
ranks generate must be exactly the full scene, each particle once."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_04658_b200 import dist as qdist
from paper_2207_04658_b200 import scenes


def test_slab_cuts_cover_on_block_planes():
    for nz, world in [(256, 2), (256, 8), (2048, 8), (66, 3)]:
        c = qdist.slab_cuts(nz, world)
        assert c[0][0] == 0 and c[-1][1] == nz and len(c) == world
        for (a, b), (a2, _) in zip(c[:-1], c[1:]):
            assert b == a2 and a % 4 == 0 and b % 4 == 0 and b > a
    w = np.zeros(64)
    w[40:] = 1.0  # all particles in the upper part: cuts balance them
    c = qdist.slab_cuts(64, 2, weights=w)
    assert c[0][1] >= 40


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    sc = scenes.small_fluid_3d()
    cuts = qdist.slab_cuts(sc.sim["grid_res"][2], world)
    uid = qdist.share_unique_id(lambda: b"\x07" * 128)
    assert uid == b"\x07" * 128
    z_lo, z_hi = qdist.rank_zrange(cuts, rank, sc.sim["dx"])
    if rank == 0:
        z_lo = -np.inf
    if rank == world - 1:
        z_hi = np.inf
    idx = np.concatenate([i for i, _ in sc.state_zrange(z_lo, z_hi, max_chunk=7000)])
    n = torch.tensor([idx.size], dtype=torch.int64)
    dist.all_reduce(n)
    gathered = [None] * world
    dist.all_gather_object(gathered, idx)
    if rank == 0:
        allidx = np.sort(np.concatenate(gathered))
        out.put((int(n.item()), bool(np.array_equal(allidx, np.arange(sc.n_particles))), sc.n_particles))
    dist.destroy_process_group()


def test_two_rank_generation_partitions_the_scene():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total, exact, n = res
    assert total == n and exact


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c4_slab_capacities_hold_every_rank(world):
    """bench.py sizes each rank's context (and its e2e host buffer) with
    dist.slab_capacity: for the weak-scaling C4 scene at 2/4/8 ranks the capacity must
    hold the rank's initial particles (upper bound from the lattice planes) with room for
    migration, although interior ranks hold MORE than n / world (the water block starts
    3 cells above the floor and ends 3 cells below the top of the z range)."""
    sc = scenes.c4(n_target=400_000_000 * world, z_extent=float(world))
    cuts = qdist.slab_cuts(sc.sim["grid_res"][2], world)
    bounds = [qdist.rank_count_bound(sc, cuts, r) for r in range(world)]
    assert sum(bounds) >= sc.n_particles
    per = sc.n_particles / world
    assert max(bounds) > per  # the round-1 sizing (n / world) was too small
    for r in range(world):
        cap = qdist.slab_capacity(sc, cuts, r)
        assert cap >= 1.2 * bounds[r], (r, cap, bounds[r])
        assert cap < 2 ** 32 - 1


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_weak_scaling_scheme_covers_the_domain(k):
    """bench.py --gpus k extends C4 k times along z; the position fields must cover
    [0, k) without saturating, with Delta unchanged (the integer next-step key needs
    Delta_x = 2^-18 on every axis) and F2's record still 8 words."""
    from paper_2207_04658_b200 import qmpm, schemes
    sc = scenes.c4(n_target=1000, z_extent=float(k))
    sch = schemes.with_domain(schemes.f2(), sc.sim)
    for f in sch["fields"]:
        if f["attr"] == "x":
            ext = sc.sim["grid_res"][f["comp"]] * sc.sim["dx"]
            assert f["range"] >= ext
            assert f["range"] * 2.0 ** -f["frac_bits"] == 2.0 ** -18
    assert qmpm.layout(sch)[1] == 8
