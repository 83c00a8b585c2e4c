"""The multi-GPU LU driver with the PRODUCT backend (CudaBackend: C-ABI on
device pointers) on the single GPU this build has:

* world size 1 over NCCL -- the production collective path;
* world size 2 over gloo with both ranks on cuda:0 (host-level collectives
  only; no kernel waits on another rank, so sharing the device is safe).

Both must reproduce the single-GPU factorization bit for bit."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from testpaths import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, case, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_2403_16013_b200 as pkg
    from paper_2403_16013_b200 import problems
    from paper_2403_16013_b200.dist import CudaBackend, Layout, TorchComm, dist_getrf

    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        n, K, k, method = case[:4]
        rk = case[4] if len(case) > 4 else "blocked"
        re, im = problems.lu_matrix(n, k, 11, populate_lower=k > 2,
                                    renorm=pkg.renorm_planes if k > 2 else None)
        dev = torch.device("cuda", 0)
        lay = Layout(n, K, world, rank)
        lr = torch.from_numpy(lay.scatter(re)).to(dev)
        li = torch.from_numpy(lay.scatter(im)).to(dev)
        piv = torch.arange(n, dtype=torch.int64, device=dev)
        dist_getrf(CudaBackend(k, method, dev, rk), TorchComm(dist), lay, k, lr, li, piv, True)
        torch.cuda.synchronize()
        objs = [None] * world
        dist.all_gather_object(objs, (rank, lr.cpu().numpy(), li.cpu().numpy(), piv.cpu().numpy()))
        if rank == 0:
            fr, fi = np.zeros_like(re), np.zeros_like(im)
            for r, a, b, _ in objs:
                L = Layout(n, K, world, r)
                L.gather_into(fr, a)
                L.gather_into(fi, b)
            f = pkg.lu_blocked(pkg.PlanarComplexMatrix(pkg.RealMatrix(re), pkg.RealMatrix(im)), K,
                               kc=pkg.KernelChoice(method=method, real_kernel=rk))
            ok = all(np.array_equal(o[3], f.pivots) for o in objs)
            ok = ok and fr.tobytes() == f.packed.re_plane.data.tobytes()
            ok = ok and fi.tobytes() == f.packed.im_plane.data.tobytes()
            q.put("ok" if ok else "mismatch")
    except Exception as e:  # pragma: no cover
        q.put(f"error rank {rank}: {e!r}")
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,backend,case", [
    (1, "nccl", (300, 64, 2, "3m")),
    (2, "gloo", (300, 64, 2, "3m")),
    (2, "gloo", (257, 48, 2, "4m")),
    (2, "gloo", (96, 32, 3, "3m")),
    (1, "nccl", (300, 64, 2, "3m", "ozaki")),
    (2, "gloo", (257, 48, 2, "4m", "ozaki")),
])
def test_dist_cuda_backend_bitwise(world, backend, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, case, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) == "ok"


def _public_worker(port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_2403_16013_b200 as pkg
    from paper_2403_16013_b200 import problems
    from paper_2403_16013_b200.dist import lu_blocked_distributed

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        re, im = problems.lu_matrix(200, 2, 5)
        fr, fi, piv = lu_blocked_distributed(re, im, 48, "3m")
        f = pkg.lu_blocked(pkg.PlanarComplexMatrix(pkg.RealMatrix(re), pkg.RealMatrix(im)), 48)
        ok = (np.array_equal(piv, f.pivots) and fr.tobytes() == f.packed.re_plane.data.tobytes()
              and fi.tobytes() == f.packed.im_plane.data.tobytes())
        q.put("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


def test_public_distributed_api_nccl():
    """lu_blocked_distributed (scatter from host, NCCL gather to rank 0)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_public_worker, args=(_free_port(), q))
    p.start()
    p.join(timeout=600)
    assert p.exitcode == 0
    assert q.get(timeout=5) == "ok"
