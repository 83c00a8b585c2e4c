"""Multi-GPU blocked LU: 1-D block-column-cyclic distribution with a panel +
pivot broadcast per step (BASELINE.json config 4).

Block column b (global columns [b*K, min((b+1)*K, n))) lives on rank
b mod P; every rank stores its blocks side by side in a local (k, n, ncols)
array per Re / Im.  Step b:

1. the owner factors the panel (``mpc_panel_factor``: recursive panel,
   interchanges applied only inside the panel) and packs rows [jb, n) of the
   panel into a contiguous buffer;
2. the panel buffer and piv[jb:jb+kw] are broadcast (NCCL over NVLink in
   production, gloo in the CPU tests);
3. every rank applies the interchanges to its other columns (LASWP), solves
   its U12 columns with L11 (right-looking TRSM) and applies the fused 3M/4M
   trailing update ``A22 -= L21 U12`` to its trailing columns.

Lookahead (depth 1): the owner of block b+1 updates that block first,
factors panel b+1 and starts its broadcast before finishing the rest of
step b's update, so panel factorization overlaps the other ranks' updates.

Every element sees exactly the operation sequence of the 1-GPU factorization
(panel chains, TRSM chains and GEMM chains are per element and independent
of the column distribution), so the distributed result is bit-identical to
``lu_blocked`` / the reference.  The backend is injected: ``CudaBackend``
(this module, C-ABI on device pointers) is the product; the CPU tests use an
oracle-backed backend to exercise the same schedule with gloo.
"""

from dataclasses import dataclass

import numpy as np


@dataclass
class PView:
    """Planar complex view: element (i, j), limb c at flat[off + c*ps + i*ld + j]."""

    re: object  # flat-addressable storage (torch tensor)
    im: object
    off: int
    ld: int
    ps: int

    def sub(self, r, c):
        return PView(self.re, self.im, self.off + r * self.ld + c, self.ld, self.ps)


class Layout:
    """Block-column-cyclic ownership and local column offsets."""

    def __init__(self, n, K, world, rank):
        self.n, self.K, self.world, self.rank = n, K, world, rank
        self.nb = (n + K - 1) // K
        self.owned = [b for b in range(self.nb) if b % world == rank]
        self.lcol = {}
        c = 0
        for b in self.owned:
            self.lcol[b] = c
            c += self.width(b)
        self.ncols = c

    def width(self, b):
        return min(self.K, self.n - b * self.K)

    def owner(self, b):
        return b % self.world

    def first_owned_after(self, b):
        for ob in self.owned:
            if ob > b:
                return ob
        return None

    def scatter(self, full):
        """Local (k, n, ncols) copy of this rank's blocks of a (k, n, n) array."""
        k, n, _ = full.shape
        out = np.empty((k, n, self.ncols))
        for b in self.owned:
            j0 = b * self.K
            out[:, :, self.lcol[b]:self.lcol[b] + self.width(b)] = full[:, :, j0:j0 + self.width(b)]
        return out

    def gather_into(self, full, local):
        for b in self.owned:
            j0 = b * self.K
            full[:, :, j0:j0 + self.width(b)] = local[:, :, self.lcol[b]:self.lcol[b] + self.width(b)]


class CudaBackend:
    """Product backend: libmpcb200 on device pointers, current torch stream.
    real_kernel="ozaki": the trailing update through the Ozaki scheme on the
    INT8 tensor cores (lu_blocked with KernelChoice(real_kernel="ozaki")) --
    column ranges of that update are independent too (right-operand grids
    per column, left-operand grids per row of L21), so the distributed
    result stays bit-identical to the 1-GPU one."""

    def __init__(self, k, method, device, real_kernel="blocked", d=None, split_bits=None):
        import torch

        from . import _lib

        self.torch = torch
        self.k = k
        self.meth = 3 if method == "3m" else 4
        self.device = device
        self.L = _lib.lib()
        self._lib = _lib
        self.ozaki = real_kernel == "ozaki"
        self.d = d if d is not None else {2: 6, 3: 8, 4: 12}[k]   # cmatrix.py:26
        self.split_bits = split_bits or 0

    def _p(self, t, off):
        return t.data_ptr() + 8 * off

    def _st(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def empty(self, shape, dtype="f64"):
        dt = self.torch.float64 if dtype == "f64" else self.torch.int64
        return self.torch.empty(shape, dtype=dt, device=self.device)

    def panel_factor(self, V, n, jb, kw, piv):
        # the C entry point takes the address of element (0, jb)
        return self._lib.check(self.L.mpc_panel_factor(
            self.k, self.meth, n, jb, kw, self._p(V.re, V.off + jb), self._p(V.im, V.off + jb),
            V.ld, V.ps, piv.data_ptr(), self._st()), "panel_factor")

    def laswp(self, V, ncols, piv, r0, r1):
        if ncols <= 0:
            return
        self._lib.check(self.L.mpc_laswp(self.k, ncols, self._p(V.re, V.off), self._p(V.im, V.off),
                                         V.ld, V.ps, piv.data_ptr(), r0, r1, self._st()), "laswp")

    def trsm(self, L11, X, kb, M):
        if M <= 0:
            return
        self._lib.check(self.L.mpc_trsm_ll_unit(
            self.k, self.meth, kb, M, self._p(L11.re, L11.off), self._p(L11.im, L11.off), L11.ld,
            L11.ps, self._p(X.re, X.off), self._p(X.im, X.off), X.ld, X.ps, self._st()), "trsm")

    def gemm_sub(self, A, B, C, m, kin, l):
        if m <= 0 or l <= 0:
            return
        if self.ozaki:
            self._lib.check(self.L.mpc_cgemm_ozaki(
                self.k, self.meth, m, kin, l, self._p(A.re, A.off), self._p(A.im, A.off), A.ld,
                A.ps, self._p(B.re, B.off), self._p(B.im, B.off), B.ld, B.ps,
                self._p(C.re, C.off), self._p(C.im, C.off), C.ld, C.ps, self.d, self.split_bits,
                1, self._st()), "cgemm_ozaki")
            return
        self._lib.check(self.L.mpc_cgemm(
            self.k, self.meth, m, kin, l, self._p(A.re, A.off), self._p(A.im, A.off), A.ld, A.ps,
            self._p(B.re, B.off), self._p(B.im, B.off), B.ld, B.ps, self._p(C.re, C.off),
            self._p(C.im, C.off), C.ld, C.ps, 1, self._st()), "cgemm")

    def pack_panel(self, loc_re, loc_im, lay, b, buf_re, buf_im):
        """rows [jb, n) of block b's local columns -> contiguous buffers."""
        jb, kw, lc = b * lay.K, lay.width(b), lay.lcol[b]
        buf_re.copy_(loc_re[:, jb:, lc:lc + kw])
        buf_im.copy_(loc_im[:, jb:, lc:lc + kw])

    # --- asynchronous panel on a high-priority side stream (lookahead) ---
    def side(self):
        if not hasattr(self, "_side"):
            self._side = self.torch.cuda.Stream(device=self.device, priority=-1)
        return self._side

    def side_context(self):
        return self.torch.cuda.stream(self.side())

    def side_wait_main(self):
        self.side().wait_stream(self.torch.cuda.current_stream(self.device))

    def main_wait_side(self):
        self.torch.cuda.current_stream(self.device).wait_stream(self.side())

    def panel_factor_meta(self, V, n, jb, kw, piv, meta):
        """Enqueue the panel on the current stream; status -> meta[kw],
        pivots -> meta[:kw] (device side, no host synchronisation)."""
        self._lib.check(self.L.mpc_panel_factor_async(
            self.k, self.meth, n, jb, kw, self._p(V.re, V.off + jb), self._p(V.im, V.off + jb),
            V.ld, V.ps, piv.data_ptr(), meta[kw:].data_ptr(), self._st()), "panel_factor")
        meta[:kw].copy_(piv[jb:jb + kw])


class _NoStream:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def dist_getrf(backend, comm, lay, k, loc_re, loc_im, piv, lookahead=True):
    """Factor the distributed matrix in place.

    loc_re / loc_im: this rank's (k, n, ncols) local blocks (contiguous,
    backend storage); piv: (n,) int64 backend array, receives all pivots.
    comm: object with broadcast(tensor, src) (torch.distributed in
    production).  Returns -1 or raises SingularMatrixError on every rank.
    """
    from .lu import SingularMatrixError

    n, K = lay.n, lay.K
    A = PView(loc_re, loc_im, 0, lay.ncols, n * lay.ncols)
    nb = lay.nb
    if nb == 0:
        return -1

    asyncp = hasattr(backend, "panel_factor_meta")

    def panel_step(b):
        """Factor panel b (owner) and start its broadcast; returns (bufs,
        works).  With an async backend the panel and the broadcast run on
        the side stream, so the caller's trailing update overlaps them."""
        jb, kw = b * K, lay.width(b)
        buf_re = backend.empty((k, n - jb, kw))
        buf_im = backend.empty((k, n - jb, kw))
        meta = backend.empty((kw + 1,), "i64")
        owner = lay.owner(b) == lay.rank
        if asyncp:
            backend.side_wait_main()
        ctx = backend.side_context() if asyncp else _NoStream()
        with ctx:
            if owner:
                V = A.sub(0, lay.lcol[b] - jb)
                if asyncp:
                    backend.panel_factor_meta(V, n, jb, kw, piv, meta)
                else:
                    st = backend.panel_factor(V, n, jb, kw, piv)
                    meta[:kw].copy_(piv[jb:jb + kw])
                    meta[kw] = st
                backend.pack_panel(loc_re, loc_im, lay, b, buf_re, buf_im)
            src = lay.owner(b)
            works = [comm.broadcast(meta, src), comm.broadcast(buf_re, src),
                     comm.broadcast(buf_im, src)]
        return (buf_re, buf_im, meta), works

    def apply_panel(b, bufs, col_lo, col_hi):
        """LASWP + TRSM + trailing update for local columns [col_lo, col_hi)
        (local indices), restricted to columns right of panel b for the
        TRSM / update; LASWP applies to the given range except the panel."""
        jb, kw = b * K, lay.width(b)
        end = jb + kw
        buf_re, buf_im, meta = bufs
        L11 = PView(buf_re, buf_im, 0, kw, (n - jb) * kw)
        # interchanges on every local column of the range except panel b itself
        pb = (lay.lcol[b], lay.lcol[b] + kw) if lay.owner(b) == lay.rank else None
        if pb is None or col_hi <= pb[0] or col_lo >= pb[1]:
            backend.laswp(A.sub(0, col_lo), col_hi - col_lo, piv, jb, end)
        else:
            backend.laswp(A.sub(0, col_lo), pb[0] - col_lo, piv, jb, end)
            backend.laswp(A.sub(0, pb[1]), col_hi - pb[1], piv, jb, end)
        # trailing columns of this range: owned blocks > b
        tb = lay.first_owned_after(b)
        if tb is None:
            return
        lo = max(col_lo, lay.lcol[tb])
        if lo >= col_hi:
            return
        M = col_hi - lo
        backend.trsm(L11, A.sub(jb, lo), kw, M)
        if end < n:
            backend.gemm_sub(L11.sub(kw, 0), A.sub(jb, lo), A.sub(end, lo), n - end, kw, M)

    # first singular column, kept on the device: no host synchronisation per
    # step (the schedule keeps running on a singular panel; the error is
    # raised once at the end with the first singular column, as lu.py:139-141
    # reports it)
    first_sing = backend.empty((1,), "i64")
    first_sing.fill_(-1)

    def check_status(b, bufs, works):
        nonlocal first_sing
        if asyncp:
            backend.main_wait_side()
        for w in works:
            if w is not None:
                w.wait()
        meta = bufs[2]
        kw = lay.width(b)
        jb = b * K
        piv[jb:jb + kw].copy_(meta[:kw])
        first_sing = first_sing.where(first_sing >= 0, meta[kw:kw + 1])

    bufs, works = panel_step(0)
    for b in range(nb):
        check_status(b, bufs, works)
        nxt = b + 1 if b + 1 < nb else None
        if nxt is not None and lookahead and lay.owner(nxt) == lay.rank:
            # update block nxt first, factor and ship panel nxt (side
            # stream), then the rest of step b overlaps it
            c0 = lay.lcol[nxt]
            c1 = c0 + lay.width(nxt)
            apply_panel(b, bufs, c0, c1)
            nbufs, nworks = panel_step(nxt)
            apply_panel(b, bufs, 0, c0)
            apply_panel(b, bufs, c1, lay.ncols)
        else:
            apply_panel(b, bufs, 0, lay.ncols)
            if nxt is not None:
                nbufs, nworks = panel_step(nxt)
        if nxt is not None:
            bufs, works = nbufs, nworks
    if asyncp:
        backend.main_wait_side()
    st = int(first_sing.item())
    if st >= 0:
        raise SingularMatrixError(st)
    return -1


class TorchComm:
    def __init__(self, dist):
        self.dist = dist

    def broadcast(self, t, src):
        return self.dist.broadcast(t, src, async_op=True)


def lu_blocked_distributed(re, im, K, method="3m", lookahead=True, real_kernel="blocked"):
    """Public multi-GPU entry point: factor a (k, n, n) host matrix over all
    ranks of the default process group (one CUDA device per rank, NCCL).
    Every rank passes the same host arrays (each copies only its own block
    columns to its device); rank 0 receives (packed_re, packed_im, pivots) as
    host arrays, the other ranks None.  Raises SingularMatrixError on every
    rank like lu_blocked."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    k, n, _ = re.shape
    dev = torch.device("cuda", torch.cuda.current_device())
    lay = Layout(n, K, world, rank)
    loc_re = torch.from_numpy(lay.scatter(re)).to(dev)
    loc_im = torch.from_numpy(lay.scatter(im)).to(dev)
    piv = torch.arange(n, dtype=torch.int64, device=dev)
    be = CudaBackend(k, method, dev, real_kernel)
    dist_getrf(be, TorchComm(dist), lay, k, loc_re, loc_im, piv, lookahead)
    return gather_factors(lay, loc_re, loc_im, piv, re.shape)


def gather_factors(lay, loc_re, loc_im, piv, shape):
    """NCCL gather of every rank's block columns to rank 0 (padded to the
    widest rank), then one D2H copy on rank 0."""
    import torch
    import torch.distributed as dist

    k, n, _ = shape
    world, rank = lay.world, lay.rank
    wmax = max(Layout(n, lay.K, world, r).ncols for r in range(world))
    out = []
    for t in (loc_re, loc_im):
        pad = torch.zeros((k, n, wmax), dtype=t.dtype, device=t.device)
        pad[:, :, :lay.ncols].copy_(t)
        bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
        dist.gather(pad, bufs, dst=0)
        out.append(bufs)
    if rank != 0:
        return None
    fr = np.empty(shape)
    fi = np.empty(shape)
    for r in range(world):
        L = Layout(n, lay.K, world, r)
        L.gather_into(fr, out[0][r][:, :, :L.ncols].cpu().numpy())
        L.gather_into(fi, out[1][r][:, :, :L.ncols].cpu().numpy())
    return fr, fi, piv.cpu().numpy()


def bench_main(args, rank, world, re0, im0, metric, workload):
    """bench.py's N > 1 leg: strong scaling of config 4 over `world` GPUs."""
    import json

    import torch
    import torch.distributed as dist

    from . import _lib

    if not dist.is_initialized():
        dist.init_process_group("nccl")
    dev = torch.device("cuda", torch.cuda.current_device())
    k, n, _ = re0.shape
    K = args.K
    lay = Layout(n, K, world, rank)
    src_re = torch.from_numpy(lay.scatter(re0)).to(dev)
    src_im = torch.from_numpy(lay.scatter(im0)).to(dev)
    loc_re, loc_im = torch.empty_like(src_re), torch.empty_like(src_im)
    piv = torch.empty(n, dtype=torch.int64, device=dev)
    be = CudaBackend(k, args.method, dev, getattr(args, "real_kernel", "blocked"))
    comm = TorchComm(dist)

    def step():
        loc_re.copy_(src_re)
        loc_im.copy_(src_im)
        piv.copy_(torch.arange(n, device=dev))
        dist_getrf(be, comm, lay, k, loc_re, loc_im, piv, lookahead=True)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = None
    if rank == 0:
        from bench import ClockSampler

        clocks = ClockSampler(dev.index)
        clocks.start()
    from . import device as _dev

    ozaki = getattr(args, "real_kernel", "blocked") == "ozaki"
    peak = _dev.int8_peak() if ozaki else _dev.fp64_peak()
    _lib.prof_enable(True, classes=["gemm"])  # the dominant kernel's launches, this rank
    l0 = _lib.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    g_ms, g_ops, g_cnt = _lib.prof_summary()["gemm"]
    _lib.prof_enable(False)
    ach = g_ops / (g_ms * 1e-3) / 1e12 if g_ms > 0 else 0.0
    roof = {"bound": "tensor" if ozaki else "fp64", "achieved": ach, "peak": peak / 1e12,
            "frac": ach * 1e12 / peak,
            "unit": "TOP/s (INT8 tensor-core ops)" if ozaki else "TFLOP/s (FP64 instr/s)",
            "traffic": None, "launches": g_cnt,
            "kernel": "ozaki_tc_kernel" if ozaki else "gemm_kernel<K=2,MODE_G3> (rank 0)",
            "peak_source": "measured on this device, this run"}
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    ms_step = float(ms.item()) / args.steps
    launches = int(_lib.launch_count() - l0)
    clk = clocks.stop() if clocks else None
    # e2e: the public multi-GPU API from host arrays (H2D scatter, factor,
    # NCCL gather, D2H on rank 0), device-timed on every rank, max over ranks
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        dist.barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        res = lu_blocked_distributed(re0, im0, K, args.method,
                                     real_kernel=getattr(args, "real_kernel", "blocked"))
        a1.record()
        torch.cuda.synchronize()
        te = torch.tensor([a0.elapsed_time(a1)], device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        same = None
        if rank == 0:
            same = bool(np.array_equal(res[2], piv.cpu().numpy()))
        e2e = {"value": 8.0 * n ** 3 / 3.0 / (float(te.item()) * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(re0.nbytes + im0.nbytes),
               "d2h_bytes_per_step": int(re0.nbytes + im0.nbytes + 8 * n),
               "ms_per_step": float(te.item()), "steps": 1, "pivots_match_device_run": same,
               "api": "paper_2403_16013_b200.dist.lu_blocked_distributed"}
    pv = [torch.empty_like(piv) for _ in range(world)]
    dist.all_gather(pv, piv)
    consistent = all(bool(torch.equal(pv[0], p)) for p in pv)
    if rank == 0:
        value = 8.0 * n ** 3 / 3.0 / (ms_step * 1e-3) / 1e9
        out = {"metric": metric, "value": value, "unit": "GFLOP/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f64 (double-double expansion)", "data": "synthetic",
               "config": {"workload": workload, "n": n, "K": K, "k": k, "method": args.method,
                          "parallelism": f"1-D block-column-cyclic over {world} GPUs, NCCL "
                                         "panel+pivot broadcast, lookahead 1"},
               "pivots_consistent_across_ranks": consistent, "clocks": clk, "e2e": e2e,
               "gpu_launches": launches, "roofline": roof, "cpu_baseline": None,
               "timing": "CUDA events per rank, max over ranks"}
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
