"""Benchmark harness on the device -- the reference's bench.py surface
(mpclu/bench.py:48-385) with a device column.

Same names and meaning as the reference: ``BenchConfig`` (bench.py:83-141),
``BenchRecord`` (bench.py:144-173), ``gen_problem`` (bench.py:176-190),
``reference_rhs`` (bench.py:199-213), ``run_bench`` (bench.py:223-280),
``run_matmul_bench`` (bench.py:283-333), ``emit_csv`` / ``read_csv``
(bench.py:351-385) and the 12 CSV columns (bench.py:48-61).  Differences,
all explicit:

* every record carries six more columns -- ``device, ngpus, gflops_conv,
  fp64_pct, pivots_equal, bwd_err`` -- written after the reference's twelve;
  ``read_csv`` accepts both layouts;
* ``reference_rhs`` and the matmul check (``_matmul_check``) run at k = 8
  (REFERENCE_K) on the device's verification kernels, as the reference
  (bench.py:199-213, 336-348);
* ``kernel`` accepts ``"b200"`` (= the EFT kernel) besides the reference's
  names; ``strassen`` is rejected as in cmatrix.KernelChoice;
* ``fp64_pct`` is the algorithmic FP64 op count of the factorization (op
  model v1) over the measured FP64 peak, for the EFT kernel;
  ``bwd_err`` is the O(n^2) normwise backward-error probe at k + 2
  components (the k = 5, 6 verification kernels for TD / QD); ``pivots_equal``
  says whether every repetition produced the same pivot vector.

No CPU fallback: every number comes from the CUDA library.
"""

import csv
import hashlib
import statistics
import time
from decimal import Decimal, localcontext
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from .cmatrix import DEFAULT_SPLITS, KernelChoice, PlanarComplexMatrix, cgemm_4m
from .expansion import PRECISIONS, REFERENCE_K, eps_for, exp_to_string
from .lu import (ComplexVector, LinearSystem, SingularMatrixError, backward_error_probe,
                 lu_blocked, lu_normal, max_rel_err, reconstruction_error, solve)
from .rmatrix import RealMatrix, mat_sub

CSV_COLUMNS = ["precision", "algorithm", "method", "kernel", "n", "K", "splits", "threads",
               "rep_median_seconds", "max_relerr", "seed", "status"]   # bench.py:48-61
EXT_COLUMNS = ["device", "ngpus", "gflops_conv", "fp64_pct", "pivots_equal", "bwd_err"]

DEFAULT_BLOCK = 16      # rgemm.py:26
DEFAULT_THRESHOLD = 32  # rgemm.py:27

# op model v1: FP64 ops per complex MAC of the trailing
# update and per panel / TRSM element update, 3M / 4M
_OPS = {2: ((93, 173), (124, 124)), 3: ((585, 833), (780, 780)), 4: ((975, 1323), (1300, 1300))}


def _resolve_k(precision):
    """bench.py:64-73"""
    if isinstance(precision, str):
        try:
            return PRECISIONS[precision.lower()]
        except KeyError:
            raise ValueError(f"unknown precision {precision!r}") from None
    k = int(precision)
    if k < 2:
        raise ValueError("precision must name dd/td/qd or give k >= 2")
    return k


def _precision_name(k):
    for name, kk in PRECISIONS.items():
        if kk == k:
            return name
    return f"k{k}"


@dataclass
class BenchConfig:
    """bench.py:83-141 (kernel default "b200": the device EFT kernel)."""

    precision: str = "dd"
    algorithm: str = "blocked"          # normal | blocked
    method: str = "3m"                  # 3m | 4m
    kernel: str = "b200"                # naive | blocked | b200 | ozaki
    n: int = 256
    seed: int = 1
    k_values: List[int] = field(default_factory=list)
    splits: Optional[int] = None
    block: int = DEFAULT_BLOCK
    threshold: int = DEFAULT_THRESHOLD
    threads: List[int] = field(default_factory=lambda: [1])
    reps: int = 3
    verify: bool = False

    def validate(self):
        k = _resolve_k(self.precision)
        if k not in (2, 3, 4):
            raise ValueError("the device kernels support k = 2, 3, 4")
        if self.algorithm not in ("normal", "blocked"):
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.n < 1:
            raise ValueError("n must be >= 1")
        if self.reps < 1:
            raise ValueError("repetitions must be >= 1")
        if self.splits is not None and self.splits < 1:
            raise ValueError("splits must be >= 1")
        for K in self.k_values:
            if not 1 <= K <= self.n:
                raise ValueError(f"K={K} outside [1, {self.n}]")
        for t in self.threads:
            if t < 1:
                raise ValueError("thread counts must be >= 1")
        if self.kernel == "strassen":
            raise ValueError("strassen is square-only in the reference and not built here")
        self.kernel_choice().validate()
        return self

    def kernel_choice(self):
        return KernelChoice(method=self.method, real_kernel=self.kernel, block=self.block,
                            threshold=self.threshold, d=self.splits)

    def sweep(self):
        """bench.py:127-137"""
        if self.algorithm == "normal":
            return [self.n]
        if self.k_values:
            return list(self.k_values)
        if self.n < 32:
            return [self.n]
        return list(range(32, self.n + 1, 32))

    def effective_splits(self, k):
        return self.splits if self.splits is not None else DEFAULT_SPLITS.get(k, 8)


@dataclass
class BenchRecord:
    """bench.py:144-173 plus the device columns (EXT_COLUMNS)."""

    precision: str
    algorithm: str
    method: str
    kernel: str
    n: int
    K: int
    splits: int
    threads: int
    rep_median_seconds: float
    max_relerr: str
    seed: int
    status: str
    run_id: str = ""
    device: str = "b200"
    ngpus: int = 1
    gflops_conv: float = float("nan")
    fp64_pct: float = float("nan")
    pivots_equal: bool = True
    bwd_err: float = float("nan")

    def row(self):
        return [self.precision, self.algorithm, self.method, self.kernel, str(self.n), str(self.K),
                str(self.splits), str(self.threads), repr(self.rep_median_seconds),
                self.max_relerr, str(self.seed), self.status]

    def ext_row(self):
        return self.row() + [self.device, str(self.ngpus), repr(self.gflops_conv),
                             repr(self.fp64_pct), str(int(self.pivots_equal)), repr(self.bwd_err)]


def reference_rhs(A, x):
    """bench.py:199-213: b := A x with every operand widened to k = 8
    (REFERENCE_K, exact), the 4M product on the k = 8 verification kernels
    (naive ≡ blocked bitwise), then truncated back to the working precision
    (truncate = the leading k limbs renormalized, rmatrix.py:75-81)."""
    if x.n != A.cols or x.k != A.k:
        raise ValueError("x does not match A")
    k, n = A.k, A.rows
    A8 = PlanarComplexMatrix(A.re_plane.promote(REFERENCE_K), A.im_plane.promote(REFERENCE_K))
    X8 = PlanarComplexMatrix(
        RealMatrix(np.ascontiguousarray(x.re.reshape(k, n, 1))).promote(REFERENCE_K),
        RealMatrix(np.ascontiguousarray(x.im.reshape(k, n, 1))).promote(REFERENCE_K))
    B8 = cgemm_4m(A8, X8, KernelChoice(method="4m", real_kernel="naive"))
    del A8
    bre = B8.re_plane.truncate(k)
    bim = B8.im_plane.truncate(k)
    return ComplexVector(bre.data.reshape(k, n), bim.data.reshape(k, n))


def _matmul_check(A, B, C):
    """bench.py:336-348: max componentwise relative error of C against the
    k = 8 product (4M, blocked) on the verification kernels."""
    A8 = PlanarComplexMatrix(A.re_plane.promote(REFERENCE_K), A.im_plane.promote(REFERENCE_K))
    B8 = PlanarComplexMatrix(B.re_plane.promote(REFERENCE_K), B.im_plane.promote(REFERENCE_K))
    R = cgemm_4m(A8, B8, KernelChoice(method="4m", real_kernel="blocked"))
    worst = 0.0
    for plane_c, plane_r in ((C.re_plane, R.re_plane), (C.im_plane, R.im_plane)):
        D = mat_sub(plane_c.promote(REFERENCE_K), plane_r)
        denom = np.maximum(np.abs(plane_r.data[0]), np.finfo(float).tiny)
        worst = max(worst, float((np.abs(D.data[0]) / denom).max()))
    return worst


def float_to_string(v, digits=17):
    """exp_to_string(Expansion.from_float(v, k), digits) (expansion.py:199-215)
    for a binary64 value: correctly rounded decimal, same formatting."""
    if v == 0.0:
        return "0.0"
    with localcontext() as ctx:
        ctx.prec = digits
        d = +Decimal(v)
    s = str(d)
    if "E" in s:
        s = s.replace("E", "e")
    elif "." not in s:
        s += ".0"
    return s


def gen_problem(n, seed, precision):
    """bench.py:176-190: Philox(seed), Re and Im U[0,1) in the leading limb,
    x_k = k + k i (k = 1..n)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    k = _resolve_k(precision)
    rng = np.random.Generator(np.random.Philox(key=np.uint64(seed)))
    re = RealMatrix.from_float64(rng.random((n, n)), k)
    im = RealMatrix.from_float64(rng.random((n, n)), k)
    A = PlanarComplexMatrix(re, im)
    x = ComplexVector.zeros(n, k)
    idx = np.arange(1, n + 1, dtype=np.float64)
    x.re[0] = idx
    x.im[0] = idx
    return LinearSystem(A=A, b=reference_rhs(A, x)), x


def _run_id(cfg, K, threads):
    return hashlib.sha1(f"{cfg!r}|{K}|{threads}|{time.time_ns()}".encode()).hexdigest()[:12]


def _factor_ops(n, K, k, method, normal):
    """Algorithmic FP64 ops of one factorization (op model v1): trailing
    updates sum over panels of M^2 K ops/cmac; panel + TRSM element updates."""
    i3 = 0 if method == "3m" else 1
    cmac, upd = _OPS[k][i3]
    ops = 0.0
    Kp = n if normal else K
    for jb in range(0, n, Kp):
        kw = min(Kp, n - jb)
        M = n - jb - kw
        ops += sum((n - j - 1) * (jb + kw - j - 1) for j in range(jb, jb + kw)) * float(upd)  # panel
        ops += M * kw * (kw - 1) / 2.0 * upd             # TRSM of U12
        ops += float(M) * M * kw * cmac                  # trailing update
    return ops


_peak_cache = {}


def _fp64_peak():
    if "fp64" not in _peak_cache:
        import torch

        _peak_cache["fp64"] = float(_lib.lib().mpc_fp64_peak(20000,
                                                             torch.cuda.current_stream().cuda_stream))
    return _peak_cache["fp64"]


def run_bench(cfg):
    """bench.py:223-280 on the device: per (K, threads) the median over reps
    of factorize + solve; singular cases are recorded and the sweep goes on."""
    cfg.validate()
    _lib.require_device()
    k = _resolve_k(cfg.precision)
    system, x_true = gen_problem(cfg.n, cfg.seed, cfg.precision)
    d = cfg.effective_splits(k)
    records = []
    for K in cfg.sweep():
        kc = cfg.kernel_choice()
        for t in cfg.threads:
            times, pivs = [], []
            status, err_str, factors, xhat = "ok", "nan", None, None
            for _ in range(cfg.reps):
                t0 = time.perf_counter()
                try:
                    if cfg.algorithm == "normal":
                        factors = lu_normal(system.A, threads=t, method=cfg.method)
                    else:
                        factors = lu_blocked(system.A, K, kc=kc, threads=t)
                    xhat = solve(factors, system.b)
                except SingularMatrixError:
                    status = "singular"
                times.append(time.perf_counter() - t0)
                if status != "ok":
                    break
                pivs.append(factors.pivots.copy())
            rec = BenchRecord(precision=_precision_name(k), algorithm=cfg.algorithm,
                              method=cfg.method, kernel=cfg.kernel, n=cfg.n, K=K, splits=d,
                              threads=t, rep_median_seconds=statistics.median(times),
                              max_relerr=err_str, seed=cfg.seed, status=status,
                              run_id=_run_id(cfg, K, t))
            if status == "ok":
                med = rec.rep_median_seconds
                rec.max_relerr = exp_to_string(max_rel_err(xhat, x_true), 17)
                rec.gflops_conv = 8.0 * cfg.n ** 3 / 3.0 / med / 1e9
                if cfg.kernel != "ozaki":
                    ops = _factor_ops(cfg.n, K, k, cfg.method, cfg.algorithm == "normal")
                    rec.fp64_pct = 100.0 * ops / med / _fp64_peak()
                rec.pivots_equal = all(np.array_equal(p, pivs[0]) for p in pivs)
                rec.bwd_err = float(backward_error_probe(factors, system.A))  # at k + 2
                if cfg.verify:
                    # bench.py:259-262: componentwise reconstruction at k + 2
                    resid = reconstruction_error(factors, system.A)
                    if resid > 64.0 * eps_for(k) * system.A.max_abs():
                        rec.status = "verify_failed"
            records.append(rec)
    return records


def run_matmul_bench(cfg, check=False):
    """bench.py:283-333: C = A B on two seeded U[0,1) matrices, median of
    reps per thread count; check=True records the componentwise maximum
    relative error against the k = 8 product (_matmul_check)."""
    cfg.validate()
    _lib.require_device()
    from .cmatrix import cgemm

    k = _resolve_k(cfg.precision)
    n = cfg.n
    rng = np.random.Generator(np.random.Philox(key=np.uint64(cfg.seed)))
    A = PlanarComplexMatrix(RealMatrix.from_float64(rng.random((n, n)), k),
                            RealMatrix.from_float64(rng.random((n, n)), k))
    B = PlanarComplexMatrix(RealMatrix.from_float64(rng.random((n, n)), k),
                            RealMatrix.from_float64(rng.random((n, n)), k))
    records = []
    d = cfg.effective_splits(k)
    for t in cfg.threads:
        kc = cfg.kernel_choice().with_threads(t)
        times, C = [], None
        for _ in range(cfg.reps):
            t0 = time.perf_counter()
            C = cgemm(A, B, kc)
            times.append(time.perf_counter() - t0)
        err_str = "nan"
        if check:
            err_str = float_to_string(_matmul_check(A, B, C), 17)
        med = statistics.median(times)
        records.append(BenchRecord(precision=_precision_name(k), algorithm="matmul",
                                   method=cfg.method, kernel=cfg.kernel, n=n, K=0, splits=d,
                                   threads=t, rep_median_seconds=med, max_relerr=err_str,
                                   seed=cfg.seed, status="ok", gflops_conv=8.0 * n ** 3 / med / 1e9))
    return records


def emit_csv(records, path, extended=True):
    """bench.py:351-357; extended=True appends EXT_COLUMNS."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_COLUMNS + (EXT_COLUMNS if extended else []))
        for rec in records:
            w.writerow(rec.ext_row() if extended else rec.row())


def read_csv(path):
    """bench.py:360-385 (either layout; run ids are not persisted)."""
    records = []
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader)
        if header not in (CSV_COLUMNS, CSV_COLUMNS + EXT_COLUMNS):
            raise ValueError("unexpected CSV header")
        for row in reader:
            rec = BenchRecord(precision=row[0], algorithm=row[1], method=row[2], kernel=row[3],
                              n=int(row[4]), K=int(row[5]), splits=int(row[6]),
                              threads=int(row[7]), rep_median_seconds=float(row[8]),
                              max_relerr=row[9], seed=int(row[10]), status=row[11])
            if len(row) > 12:
                rec.device, rec.ngpus = row[12], int(row[13])
                rec.gflops_conv, rec.fp64_pct = float(row[14]), float(row[15])
                rec.pivots_equal, rec.bwd_err = bool(int(row[16])), float(row[17])
            records.append(rec)
    return records
