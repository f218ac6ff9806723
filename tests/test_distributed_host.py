"""CPU tests of the slab decomposition's host side (no GPU): the partition rule
(ipmg_partition, the same function ipmg_create uses) and the multi-process
bootstrap of the NCCL communicator through torch.distributed, run with the
gloo backend at world size 2."""
import os
import socket

import pytest

ipmg = pytest.importorskip("paper_2405_18982_b200.ipmg")


def _layers(dim, cc, l):
    return cc[dim - 1] << l


@pytest.mark.parametrize("dim,cc,nl", [(2, (2, 2), 10), (3, (2, 2, 2), 6), (3, (2, 2, 1), 8)])
@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
def test_partition_tiles_every_level(dim, cc, nl, nranks):
    for l in range(nl):
        parts = [ipmg.partition(dim, cc, nl, nranks, r, l) for r in range(nranks)]
        ng = _layers(dim, cc, l)
        assert all(p[3] == ng for p in parts)
        d = parts[0][0]
        assert all(p[0] == d for p in parts)
        if nranks == 1:
            assert parts[0] == (1, 0, ng, ng)
        elif d:
            # contiguous, ordered, even slabs of >= 2 layers covering the level
            z = 0
            for p in parts:
                assert p[1] == z and p[2] >= 2 and p[2] % 2 == 0 and p[1] % 2 == 0
                z += p[2]
            assert z == ng
            assert ng % (2 * nranks) == 0
        else:
            assert all(p[1] == 0 and p[2] == ng for p in parts)
            assert l == 0 or ng % (2 * nranks) != 0
        # distributed levels form a suffix of the hierarchy
        if l >= 1 and d == 0:
            assert all(ipmg.partition(dim, cc, nl, nranks, 0, m)[0] == 0 for m in range(l))


def test_partition_c4_layers_per_rank():
    """C4 (256x256x128 cells, T_0 = 2x2x1, 8 levels) on 8 GPUs
    distributes the levels with 128/64/32/16 z-layers as 16/8/4/2 per rank."""
    got = [ipmg.partition(3, (2, 2, 1), 8, 8, 0, l)[:3] for l in range(8)]
    assert [g[2] for g in got if g[0]] == [2, 4, 8, 16]
    assert [l for l in range(8) if got[l][0]] == [4, 5, 6, 7]


def test_partition_rejects_bad_args():
    with pytest.raises(ipmg.IpmgError):
        ipmg.partition(4, (2, 2, 2), 3, 1, 0, 0)
    with pytest.raises(ipmg.IpmgError):
        ipmg.partition(2, (2, 2), 3, 2, 2, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the unique-id broadcast of Comm.from_torch_distributed, with a fixed id
        uid = bytes(range(128)) if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        # every rank computes its slab of C2's finest level and gathers the others'
        mine = [ipmg.partition(2, (2, 2), 10, world, rank, l) for l in range(10)]
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        q.put((rank, obj[0], allp))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_bootstrap_and_partition():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert out[0][1] == out[1][1] == bytes(range(128))
    allp = out[0][2]
    assert allp == out[1][2]
    for l in range(10):
        d0, d1 = allp[0][l], allp[1][l]
        if d0[0]:
            assert d0[1] == 0 and d1[1] == d0[2] and d0[2] + d1[2] == d0[3]
        else:
            assert d0 == d1


def test_partition_min_local_dofs_replicates_coarse_levels():
    """C2 (2D k=7, 10 levels) on 8 ranks with a 1M-dof floor: only the levels
    where every rank keeps >= 2^20 dofs are distributed (9 and 8), a suffix of
    the hierarchy; without the floor levels 3..9 are."""
    d0 = [ipmg.partition(2, (2, 2), 10, 8, 0, l, 7, 0)[0] for l in range(10)]
    d1 = [ipmg.partition(2, (2, 2), 10, 8, 0, l, 7, 1 << 20)[0] for l in range(10)]
    assert d0 == [0, 0, 0, 1, 1, 1, 1, 1, 1, 1]
    assert d1 == [0, 0, 0, 0, 0, 0, 0, 0, 1, 1]
