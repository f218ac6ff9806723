"""Multi-process NCCL path (the 8-GPU slab decomposition of C4): two
processes, one GPU each, NCCL communicator from the torch.distributed group (the bench's
setup), against the serial library on rank 0's GPU.  Bit-identical operator, smoother
step and V-cycle (the distributed kernels compute every straddling patch from identical
ghost data), same CG iteration count and solution to 1e-12.

Needs >= 2 visible GPUs (skipped otherwise: the development boxes have one; the driver's
multi-GPU runs have eight).  The in-process team (tests/test_gpu_distributed.py) covers
the same kernels on one GPU.
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORLD = 2
CASES = {"d3k4": (3, 4, 4, None), "d3k3box": (3, 3, 4, (2, 2, 1)), "d2k5": (2, 5, 5, None)}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slice(h_serial, h, level):
    d, zoff, nglob = h.level_partition(level)
    n_loc = h.ndofs(level)
    if not d:
        return 0, n_loc
    per_layer = h_serial.ndofs(level) // nglob
    return zoff * per_layer, n_loc


def _worker(rank, port, case, outdir):
    import torch.distributed as dist
    from paper_2405_18982_b200 import ipmg
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    dim, k, nl, coarse = CASES[case]
    comm = ipmg.Comm.from_torch_distributed(rank)
    h = ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=ipmg.FP32, device=rank, comm=comm)
    hs = ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=ipmg.FP32, device=rank)   # serial
    L = nl - 1
    dev = torch.device("cuda", rank)
    g = torch.Generator().manual_seed(123)
    res = {}
    n = hs.ndofs(L)
    x64 = (torch.rand(n, dtype=torch.float64, generator=g) * 2 - 1).to(dev)
    b32 = (torch.rand(n, dtype=torch.float64, generator=g) * 2 - 1).float().to(dev)
    o, m = _slice(hs, h, L)
    # operator (fp64)
    y = torch.empty_like(x64)
    hs.vmult(L, x64, y)
    yl = torch.empty(m, dtype=torch.float64, device=dev)
    h.vmult(L, x64[o:o + m].contiguous(), yl)
    res["vmult"] = bool(torch.equal(yl, y[o:o + m]))
    # smoothing step (fp32)
    xs = x64.float()
    xl = xs[o:o + m].clone()
    hs.smooth(L, xs, b32)
    h.smooth(L, xl, b32[o:o + m].contiguous())
    res["smooth"] = bool(torch.equal(xl, xs[o:o + m]))
    # V-cycle
    z = torch.empty_like(x64)
    hs.vcycle(x64, z)
    zl = torch.empty(m, dtype=torch.float64, device=dev)
    h.vcycle(x64[o:o + m].contiguous(), zl)
    res["vcycle"] = bool(torch.equal(zl, z[o:o + m]))
    # CG on f == 1
    bb = torch.empty(n, dtype=torch.float64, device=dev)
    hs.rhs(L, bb)
    xx = torch.empty_like(bb)
    rs = hs.cg_solve(bb, xx)
    xd = torch.empty(m, dtype=torch.float64, device=dev)
    rd = h.cg_solve(bb[o:o + m].contiguous(), xd)
    res["cg_its"] = (rs["iterations"], rd["iterations"])
    res["cg_err"] = float((xd - xx[o:o + m]).abs().max() / xx.abs().max())
    torch.cuda.synchronize()
    torch.save(res, os.path.join(outdir, "rank%d.pt" % rank))
    h.close()
    hs.close()
    comm.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", list(CASES))
def test_two_process_nccl_matches_serial(case, tmp_path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < WORLD:
        pytest.skip("needs %d GPUs" % WORLD)
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(_free_port(), case, str(tmp_path)), nprocs=WORLD, start_method="spawn")
    for r in range(WORLD):
        res = torch.load(tmp_path / ("rank%d.pt" % r))
        assert res["vmult"] and res["smooth"] and res["vcycle"], (r, res)
        assert res["cg_its"][0] == res["cg_its"][1], (r, res)
        assert res["cg_err"] <= 1e-12, (r, res)
