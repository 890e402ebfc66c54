"""Host-side logic of the slab decomposition for one-process-per-GPU runs
(DESIGN.md §9): slab cuts, per-rank scene generation and the NCCL
unique-id handshake over torch.distributed.  No arithmetic of the method: the
exact particle ownership is decided on the device (qmpm_create_slab routes any
particle of an adjacent slab to its owner during the first step)."""
from __future__ import annotations

import numpy as np


def slab_cuts(nz: int, world: int, weights=None):
    """World slabs of whole 4-cell block planes covering [0, nz).  With `weights`
    (particles per cell plane, length nz) the cuts balance the particle count;
    otherwise the planes are split evenly."""
    nb = (nz + 3) // 4
    if world > nb:
        raise ValueError(f"{world} slabs need at least {world} block planes (nz={nz})")
    if weights is None:
        edges = [round(i * nb / world) for i in range(world + 1)]
    else:
        w = np.asarray(weights, np.float64)
        wb = np.add.reduceat(w, np.arange(0, nz, 4))
        c = np.concatenate([[0.0], np.cumsum(wb)])
        edges = [0]
        for i in range(1, world):
            e = int(np.searchsorted(c, c[-1] * i / world))
            edges.append(min(max(e, edges[-1] + 1), nb - (world - i)))
        edges.append(nb)
    cuts = [(4 * a, min(4 * b, nz)) for a, b in zip(edges[:-1], edges[1:])]
    return cuts


def rank_zrange(cuts, rank, dx):
    """The z interval (world units) of the particles a rank owns: base cell
    floor(z / dx - 1/2) in its planes [z0, z1), i.e. z in [(z0 + 1/2) dx, (z1 + 1/2) dx)
    (P:561's base cell), so the first step migrates only the float-rounding strays at
    the faces instead of half a cell plane (which overflowed the default migration
    buffer at 4 slabs of 25M particles)."""
    z0, z1 = cuts[rank]
    return (z0 + 0.5) * dx, (z1 + 0.5) * dx


def rank_count_bound(scene, cuts, rank):
    """Upper bound on the particles rank `rank` receives from load_slab (the lattice
    planes within 0.3 spacings of its z range: Scene.zrange_runs, a superset of the
    jittered positions) -- host arithmetic on the lattice only, no particle is generated."""
    z_lo, z_hi = rank_zrange(cuts, rank, scene.sim["dx"])
    if rank == len(cuts) - 1:
        z_hi = float("inf")
    if rank == 0:
        z_lo = float("-inf")
    return sum(c for _, c in scene.zrange_runs(z_lo, z_hi))


def slab_capacity(scene, cuts, rank, headroom=0.25, extra=65536):
    """max_particles of a rank's slab context: its initial count bound plus room for the
    particles that migrate in (the bench's sizing; tests/test_dist_host.py checks it
    against the per-rank bounds of C4 at 2, 4 and 8 ranks)."""
    per = scene.n_particles / len(cuts)
    return int(max(per, rank_count_bound(scene, cuts, rank)) * (1.0 + headroom)) + extra


def share_unique_id(uid_fn, group=None):
    """Rank 0 creates an id with uid_fn(); every rank returns it (torch.distributed)."""
    import torch.distributed as dist
    obj = [uid_fn() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def load_slab(sim, scene, cuts, rank, device="cuda", track_ids=True):
    """Generate this rank's particles (device-side, chunked) and hand them to the
    slab context; ids are the particles' global indices in the scene."""
    import torch
    z_lo, z_hi = rank_zrange(cuts, rank, scene.sim["dx"])
    if rank == len(cuts) - 1:
        z_hi = float("inf")
    if rank == 0:
        z_lo = float("-inf")
    first = True
    ids = []
    n = 0
    for idx, st in scene.state_zrange(z_lo, z_hi, backend="torch", device=device):
        if first:
            sim.set_state(st)
            first = False
        else:
            sim.append_state(st)
        ids.append(idx.to(torch.int32))
        n += st.shape[0]
        torch.cuda.current_stream().synchronize()
    if first:
        sim.set_state(torch.zeros((0, scene.n_scalars), dtype=torch.float32, device=device))
    if track_ids and n:
        sim.set_ids(torch.cat(ids))
    return n
