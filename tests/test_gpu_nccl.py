"""The NCCL transport of the slab decomposition: two processes, one GPU
each, z slabs exchanging ghost planes, velocity planes and migration buffers with
ncclSend/ncclRecv (fixed sizes) and the status all-reduce.  Skipped below 2 visible GPUs
(the driver's test box has one; the in-process transport of tests/test_gpu_slab.py runs
the same phases there).  Checks: every particle exactly once after 10 steps, and the
aggregates of the 2-rank run within 1e-3 of one context (P3)."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2207_04658_b200 import scenes, schemes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2207_04658_b200 import dist as qdist, qmpm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    sc, sch = scenes.small_fluid_3d(), schemes.f2()
    cuts = qdist.slab_cuts(sc.sim["grid_res"][2], world)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        sim = qmpm.Sim(sc.sim, sch, sc.n_particles, flags=qmpm.TRACK_IDS, stream=stream,
                       slab=(world, rank, cuts[rank][0], cuts[rank][1]))
        sim.connect_nccl(qdist.share_unique_id(qmpm.get_unique_id))
        qdist.load_slab(sim, sc, cuts, rank)
        sim.step(10)
        n = sim.stats().n_particles
        w = np.zeros((n, sim.W), np.uint32)
        ids = np.zeros(n, np.uint32)
        sim.read_state(words=w, ids=ids, capacity=n)
        sim.close()
    got = [None] * world
    dist.all_gather_object(got, (w, ids))
    if rank == 0:
        q.put(got)
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_rank_nccl_matches_one_context():
    import torch.multiprocessing as mp
    from paper_2207_04658_b200 import qmpm
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = np.concatenate([g[0] for g in got])
    ids = np.concatenate([g[1] for g in got])
    sc, sch = scenes.small_fluid_3d(), schemes.f2()
    assert np.array_equal(np.sort(ids), np.arange(sc.n_particles))
    st0 = sc.state()
    one = qmpm.Sim(sc.sim, sch, st0.shape[0])
    one.set_state(torch.from_numpy(st0).cuda())
    one.step(10)
    w1 = np.zeros((st0.shape[0], one.W), np.uint32)
    one.read_state(words=w1)
    one.close()
    ke_g, com_g = oracle.aggregates(sc.sim, oracle.decode_state(sch, w))
    ke_1, com_1 = oracle.aggregates(sc.sim, oracle.decode_state(sch, w1))
    assert abs(ke_g - ke_1) <= 1e-3 * abs(ke_1)
    assert np.all(np.abs(com_g - com_1) <= 1e-3 * np.abs(com_1))


def test_one_rank_nccl_path_matches_oracle():
    """The NCCL code path on ONE GPU: a one-rank slab context (a single-rank NCCL
    communicator is valid) loads NCCL, initialises the communicator, agrees on the
    migration capacity by the connect-time all-reduce and runs the slab phases with the
    per-step status all-reduce (no neighbour transfers).  One step meets the P2 bar
    against the fp64 oracle; ten more keep every particle."""
    from paper_2207_04658_b200 import qmpm
    from test_gpu_step import REL, dev, scales
    sc, sch = scenes.small_fluid_3d(), schemes.f2()
    w0, _ = oracle.encode_state(sch, sc.state())
    w_in, _ = oracle.run(sc.sim, sch, w0, 1, 10)
    o_pre, _, _ = oracle.step(sc.sim, sch, w_in, 11)
    n = w_in.shape[0]
    nz = sc.sim["grid_res"][2]
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        sim = qmpm.Sim(sc.sim, sch, n, flags=qmpm.TRACK_IDS | qmpm.DEBUG_PREENCODE, stream=stream,
                       slab=(1, 0, 0, nz))
        sim.connect_nccl(qmpm.get_unique_id())
        sim.set_words(dev(w_in), 10)
        sim.set_ids(dev(np.arange(n, dtype=np.uint32)))
        sim.step(1)
        m = sim.stats().n_particles
        pre = np.zeros((m, sim.n_scalars), np.float32)
        ids = np.zeros(m, np.uint32)
        sim.read_state(ids=ids, capacity=m)
        sim.read_debug(pre)
        sim.step(10)
        st = sim.stats()
        sim.close()
    assert m == n and st.n_particles == n and st.step == 21
    pre = pre[np.argsort(ids)]
    s_h = scales(sc.sim, o_pre, oracle.decode_state(sch, w_in))
    err = np.abs(pre.astype(np.float64) - o_pre) / np.maximum(np.abs(o_pre), s_h)
    assert err.max() <= REL, err.max(axis=0)
