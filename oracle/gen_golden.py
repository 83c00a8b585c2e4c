"""Generate golden vectors by running the UNMODIFIED reference (mpclu).

TEST INFRASTRUCTURE ONLY.  Imports the reference read-only from
/root/reference/pkg/src (numba JIT cache redirected to a writable dir) and
writes fixtures under tests/golden/.  The fixtures pin both the CPU oracle
(tests/test_oracle_golden.py, CPU) and the CUDA path (tests/test_gpu_*.py).
/root/reference does not exist on the GPU box, so everything the GPU tests
need is committed as these files.

    python oracle/gen_golden.py small        # scalar / small matrix vectors (npz)
    python oracle/gen_golden.py cfg0 cfg1    # BASELINE configs 0 and 1 (digests)
    python oracle/gen_golden.py cfg2         # config 2, n=4096 DD LU (~3 min)
    python oracle/gen_golden.py cfg3         # config 3, TD/QD n=2048 LU (long)
    python oracle/gen_golden.py cfg2_4m ill  # config 2 in 4M; ill-conditioned n=4096
"""

import hashlib
import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")

import numpy as np  # noqa: E402

import mpclu  # noqa: E402
from mpclu import _kernels as K  # noqa: E402
from mpclu import (  # noqa: E402
    KernelChoice,
    PlanarComplexMatrix,
    RealMatrix,
    cgemm,
    lu_blocked,
    lu_normal,
    solve,
    trsm_unit_lower,
    ComplexVector,
)
from mpclu.expansion import renormalize  # noqa: E402

from paper_2403_16013_b200 import problems  # noqa: E402

THREADS = os.cpu_count() or 8


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def ref_renorm_planes(R):
    K.renorm_planes(R, R.shape[0])
    return R


def rand_exp(rng, k, span=0):
    comps = [rng.uniform(-1.0, 1.0) * 2.0 ** span]
    for i in range(1, k):
        comps.append(rng.uniform(-1.0, 1.0) * abs(comps[0]) * 2.0 ** (-52 * i))
    return renormalize(comps, k).components


def pc(re, im):
    return PlanarComplexMatrix(RealMatrix(re), RealMatrix(im))


def meta():
    import numba

    return {
        "reference": "mpclu " + mpclu.__version__,
        "numba": numba.__version__,
        "numpy": np.__version__,
        "generated": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }


# --------------------------------------------------------------------- small

def gen_small():
    rng = np.random.default_rng(20240801)
    out = {}
    # EFTs on random pairs with varied exponents, plus hand cases
    a = rng.uniform(-1, 1, 2000) * 2.0 ** rng.integers(-60, 60, 2000)
    b = rng.uniform(-1, 1, 2000) * 2.0 ** rng.integers(-60, 60, 2000)
    a = np.concatenate([a, [2.0 ** 53, 1 + 2 ** -27, 0.1, 0.0, -0.0, 1.0]])
    b = np.concatenate([b, [1.0, 1 + 2 ** -27, 0.1, -0.0, 0.0, -1.0]])
    ts = np.array([K.two_sum(x, y) for x, y in zip(a, b)])
    tp = np.array([K.two_prod(x, y) for x, y in zip(a, b)])
    out["eft_a"], out["eft_b"], out["two_sum"], out["two_prod"] = a, b, ts, tp

    # renorm on raw term lists (lengths up to the QD mul list), incl. adversarial
    for k in (2, 3, 4):
        raws, outs = [], []
        for m in range(1, 20):
            for _ in range(40):
                span = rng.integers(0, 3)
                if span == 0:
                    raw = rng.uniform(-1, 1, m) * 2.0 ** rng.integers(-150, 5, m)
                elif span == 1:
                    base = rng.uniform(-1, 1)
                    raw = base * 2.0 ** (-53 * np.arange(m)) * rng.uniform(-1, 1, m)
                    raw[rng.integers(0, m)] *= -1
                else:
                    raw = np.round(rng.uniform(-4, 4, m)) * 2.0 ** rng.integers(-3, 3, m)
                    if m > 1:
                        raw[-1] = -raw[0]
                raws.append(np.pad(raw, (0, 19 - m)))
                outs.append(K.renorm1(raw.copy(), k))
        special = [[0.0, -0.0], [-0.0, 0.0, 1.0], [1.0, -1.0, 0.5], [1.0, -1.0],
                   [2.0 ** 57, -16.0], [1.0, 2.0 ** -53], [1.0, -(2.0 ** -54), 2.0 ** -108],
                   [-0.0, -0.0, -0.0], [3.0, -3.0, -0.0, 0.0]]
        for raw in special:
            raw = np.array(raw, dtype=np.float64)
            raws.append(np.pad(raw, (0, 19 - raw.shape[0])))
            outs.append(K.renorm1(raw.copy(), k))
        lens = [m for m in range(1, 20) for _ in range(40)] + [len(s) for s in special]
        out[f"renorm_raw_k{k}"] = np.array(raws)
        out[f"renorm_len_k{k}"] = np.array(lens, dtype=np.int64)
        out[f"renorm_out_k{k}"] = np.array(outs)

    # expansion ops and complex scalar cores
    for k in (2, 3, 4):
        N = 300
        xs = np.array([rand_exp(rng, k, rng.integers(-3, 4)) for _ in range(N)])
        ys = np.array([rand_exp(rng, k, rng.integers(-3, 4)) for _ in range(N)])
        ys[0] = xs[0]          # exact cancellation
        ys[1] = -xs[1]
        ys[2] = 0.0
        out[f"x_k{k}"], out[f"y_k{k}"] = xs, ys
        out[f"add_k{k}"] = np.array([K.exp_add1(x, y, k) for x, y in zip(xs, ys)])
        out[f"sub_k{k}"] = np.array([K.exp_sub1(x, y, k) for x, y in zip(xs, ys)])
        out[f"mul_k{k}"] = np.array([K.exp_mul1(x, y, k) for x, y in zip(xs, ys)])
        dv = ys[::-1].copy()
        dv[dv[:, 0] == 0.0] = xs[0]
        out[f"divisor_k{k}"] = dv
        out[f"div_k{k}"] = np.array([K.exp_div1(x, y, k) for x, y in zip(xs, dv)])
        # complex: a = (x, y), b = (y[::-1], x[::-1])
        c3r, c3i, c4r, c4i, cdr, cdi = [], [], [], [], [], []
        for i in range(N):
            ar, ai = xs[i], ys[i]
            br, bi = ys[N - 1 - i], xs[N - 1 - i]
            outs = [np.empty(k) for _ in range(2)]
            s = [np.empty(k) for _ in range(3)]
            buf = np.empty(K.scratch_len(k))
            K.cmul_3m_core(ar, ai, br, bi, outs[0], outs[1], s[0], s[1], s[2], buf, k)
            c3r.append(outs[0].copy()); c3i.append(outs[1].copy())
            K.cmul_4m_core(ar, ai, br, bi, outs[0], outs[1], s[0], s[1], s[2], buf, k)
            c4r.append(outs[0].copy()); c4i.append(outs[1].copy())
            K.cdiv_core(ar, ai, br, bi, outs[0], outs[1], s[0], s[1], s[2], buf, k)
            cdr.append(outs[0].copy()); cdi.append(outs[1].copy())
        out[f"cmul3_k{k}"] = np.array([c3r, c3i])
        out[f"cmul4_k{k}"] = np.array([c4r, c4i])
        out[f"cdiv_k{k}"] = np.array([cdr, cdi])

    # matrices
    def rmat(r, c, k):
        return mpclu.rmatrix.random_matrix(r, c, k, rng).data

    for k in (2, 3, 4):
        A, B = rmat(9, 11, k), rmat(9, 11, k)
        out[f"madd_A_k{k}"], out[f"madd_B_k{k}"] = A, B
        out[f"madd_k{k}"] = mpclu.mat_add(RealMatrix(A), RealMatrix(B)).data
        out[f"msub_k{k}"] = mpclu.mat_sub(RealMatrix(A), RealMatrix(B)).data
        R = rng.uniform(-1, 1, (k, 6, 7)) * 2.0 ** (-40 * np.arange(k))[:, None, None]
        out[f"rnp_in_k{k}"] = R.copy()
        out[f"rnp_out_k{k}"] = ref_renorm_planes(R.copy())
        for (m, n, l) in ((7, 5, 6), (16, 16, 16), (33, 17, 20)):
            tag = f"k{k}_{m}x{n}x{l}"
            A, B = rmat(m, n, k), rmat(n, l, k)
            out[f"rg_A_{tag}"], out[f"rg_B_{tag}"] = A, B
            out[f"rg_C_{tag}"] = mpclu.rgemm_naive(RealMatrix(A), RealMatrix(B)).data
            Ar, Ai, Br, Bi = rmat(m, n, k), rmat(m, n, k), rmat(n, l, k), rmat(n, l, k)
            out[f"cg_Ar_{tag}"], out[f"cg_Ai_{tag}"] = Ar, Ai
            out[f"cg_Br_{tag}"], out[f"cg_Bi_{tag}"] = Br, Bi
            for meth in ("3m", "4m"):
                C = cgemm(pc(Ar, Ai), pc(Br, Bi), KernelChoice(method=meth))
                out[f"cg_{meth}_{tag}"] = np.array([C.re_plane.data, C.im_plane.data])

    # LU (lu_panel / trsm / cgemm / mat_sub through the real driver)
    for k in (2, 3, 4):
        for n in (24, 37):
            tag = f"k{k}_n{n}"
            re, im = rmat(n, n, k), rmat(n, n, k)
            re[0] -= 0.5
            im[0] -= 0.5
            out[f"lu_re_{tag}"], out[f"lu_im_{tag}"] = re, im
            for meth in ("3m", "4m"):
                for Kp in (n, 8, 5):
                    if Kp == n:
                        f = lu_normal(pc(re, im), method=meth)
                    else:
                        f = lu_blocked(pc(re, im), Kp, kc=KernelChoice(method=meth))
                    key = f"lu_{meth}_K{Kp if Kp != n else 'n'}_{tag}"
                    out[key] = np.array([f.packed.re_plane.data, f.packed.im_plane.data])
                    out[key + "_piv"] = f.pivots
                    br, bi = rmat(n, 1, k)[:, :, 0], rmat(n, 1, k)[:, :, 0]
                    out[key + "_b"] = np.array([br, bi])
                    x = solve(f, ComplexVector(br, bi))
                    out[key + "_x"] = np.array([x.re, x.im])
        # TRSM
        Kt, M = 13, 9
        L = PlanarComplexMatrix.identity(Kt, k)
        L.re_plane.data[0] += np.tril(rng.uniform(-1, 1, (Kt, Kt)), -1)
        L.im_plane.data[0] += np.tril(rng.uniform(-1, 1, (Kt, Kt)), -1)
        A12 = pc(rmat(Kt, M, k), rmat(Kt, M, k))
        out[f"trsm_L_k{k}"] = np.array([L.re_plane.data, L.im_plane.data])
        out[f"trsm_A_k{k}"] = np.array([A12.re_plane.data, A12.im_plane.data])
        for meth in ("3m", "4m"):
            X = trsm_unit_lower(L, A12, method=meth)
            out[f"trsm_{meth}_k{k}"] = np.array([X.re_plane.data, X.im_plane.data])

    # singular cases (lu.py:32-35; test_lu.py:193-204)
    base = np.array([[1.0, 2.0, 1.0], [2.0, 4.0, 0.0], [3.0, 6.0, 2.0]])
    out["sing_dep"] = base
    try:
        lu_normal(pc(RealMatrix.from_float64(base, 2).data, np.zeros((2, 3, 3))))
        out["sing_dep_col"] = np.array(-1)
    except mpclu.SingularMatrixError as e:
        out["sing_dep_col"] = np.array(e.column)

    path = os.path.join(GOLD, "small.npz")
    np.savez_compressed(path, **out)
    with open(os.path.join(GOLD, "small.meta.json"), "w") as fh:
        json.dump(meta(), fh, indent=1)
    print("wrote", path, os.path.getsize(path), "bytes")


# ------------------------------------------------------------- configs 0-3

def _lu_record(re, im, K, meth, b=None):
    A = pc(re, im)
    t0 = time.perf_counter()
    if K == re.shape[1]:
        f = lu_normal(A, threads=THREADS, method=meth)
    else:
        f = lu_blocked(A, K, kc=KernelChoice(method=meth), threads=THREADS)
    dt = time.perf_counter() - t0
    rec = {
        "K": int(K), "method": meth, "seconds": dt, "threads": THREADS,
        "digest": digest(f.packed.re_plane.data, f.packed.im_plane.data),
        "digest_re": digest(f.packed.re_plane.data),
        "pivots": [int(p) for p in f.pivots],
        "u00": [f.packed.re_plane.data[:, 0, 0].tolist(), f.packed.im_plane.data[:, 0, 0].tolist()],
    }
    if b is not None:
        t0 = time.perf_counter()
        x = solve(f, ComplexVector(b[0], b[1]))
        rec["solve_seconds"] = time.perf_counter() - t0
        xt = ComplexVector(*problems.x_true(re.shape[1], re.shape[0]))
        rec["fwd_err"] = float(mpclu.max_rel_err(x, xt).to_float())
        rec["x_digest"] = digest(x.re, x.im)
    return rec, f


def rhs(re, im):
    """b = cgemm_4m(A, x_true) at working precision (naive kernel)."""
    k, n, _ = re.shape
    xr, xi = problems.x_true(n, k)
    X = pc(xr.reshape(k, n, 1).copy(), xi.reshape(k, n, 1).copy())
    B = cgemm(pc(re, im), X, KernelChoice(method="4m", real_kernel="naive", threads=THREADS))
    return np.array([B.re_plane.data[:, :, 0], B.im_plane.data[:, :, 0]])


def gen_cfg0():
    res = {"meta": meta(), "cases": []}
    n, k = 128, 2
    for seed in (1, 2, 3):
        re, im = problems.lu_matrix(n, k, seed)
        b = rhs(re, im)
        for meth in ("3m", "4m"):
            for K in (n, 32):
                rec, f = _lu_record(re, im, K, meth, b)
                rec.update(seed=seed, n=n, k=k, b_digest=digest(b))
                if seed == 1 and meth == "3m":
                    np.save(os.path.join(GOLD, f"cfg0_s1_3m_K{K}.npy"),
                            np.array([f.packed.re_plane.data, f.packed.im_plane.data]))
                res["cases"].append(rec)
                print("cfg0", seed, meth, K, rec["seconds"])
    with open(os.path.join(GOLD, "cfg0.json"), "w") as fh:
        json.dump(res, fh)


def gen_cfg1():
    res = {"meta": meta(), "cases": []}
    n, k = 1024, 2
    a, b = problems.gemm_inputs(n, k, 1, ref_renorm_planes)
    res["input_digest"] = digest(a[0], a[1], b[0], b[1])
    for meth in ("3m", "4m"):
        t0 = time.perf_counter()
        C = cgemm(pc(*a), pc(*b), KernelChoice(method=meth, real_kernel="blocked", threads=THREADS))
        dt = time.perf_counter() - t0
        res["cases"].append({
            "method": meth, "seconds": dt, "threads": THREADS, "n": n, "k": k, "seed": 1,
            "digest": digest(C.re_plane.data, C.im_plane.data),
            "row0": [C.re_plane.data[:, 0, :8].tolist(), C.im_plane.data[:, 0, :8].tolist()],
        })
        print("cfg1", meth, dt)
    with open(os.path.join(GOLD, "cfg1.json"), "w") as fh:
        json.dump(res, fh)


def gen_cfg2():
    res = {"meta": meta(), "cases": []}
    n, k, K = 4096, 2, 256
    re, im = problems.lu_matrix(n, k, 1)
    res["input_digest"] = digest(re, im)
    b = rhs(re, im)
    rec, f = _lu_record(re, im, K, "3m", b)
    rec.update(seed=1, n=n, k=k, b_digest=digest(b))
    res["cases"].append(rec)
    print("cfg2", rec["seconds"], rec.get("solve_seconds"))
    with open(os.path.join(GOLD, "cfg2.json"), "w") as fh:
        json.dump(res, fh)


def gen_cfg2_4m():
    """Adds the 4M factorization of the config-2 input to cfg2.json."""
    path = os.path.join(GOLD, "cfg2.json")
    res = json.load(open(path))
    if any(c["method"] == "4m" for c in res["cases"]):
        return
    n, k, K = 4096, 2, 256
    re, im = problems.lu_matrix(n, k, 1)
    assert digest(re, im) == res["input_digest"]
    b = rhs(re, im)
    rec, f = _lu_record(re, im, K, "4m", b)
    rec.update(seed=1, n=n, k=k, b_digest=digest(b))
    res["cases"].append(rec)
    print("cfg2 4m", rec["seconds"], rec.get("solve_seconds"))
    with open(path, "w") as fh:
        json.dump(res, fh)


def gen_ill(n=4096, K=256):
    """Config 4's ill-conditioned input (row i scaled by 10^(-12 i/n)) at a
    size the reference factors in minutes: pivots, plane digests, solve."""
    res = {"meta": meta(), "cases": []}
    k = 2
    re, im = problems.lu_matrix(n, k, 1, ill_conditioned=True)
    res["input_digest"] = digest(re, im)
    b = rhs(re, im)
    for meth in ("3m",):
        rec, f = _lu_record(re, im, K, meth, b)
        rec.update(seed=1, n=n, k=k, b_digest=digest(b), ill_conditioned=True)
        rec["digest_planes"] = [digest(f.packed.re_plane.data[c]) for c in range(k)] + \
            [digest(f.packed.im_plane.data[c]) for c in range(k)]
        res["cases"].append(rec)
        print("ill", n, meth, rec["seconds"], rec.get("solve_seconds"), flush=True)
    with open(os.path.join(GOLD, f"ill_n{n}.json"), "w") as fh:
        json.dump(res, fh)


def gen_cfg3(n=2048, K=128):
    path = os.path.join(GOLD, f"cfg3_n{n}.json")
    res = {"meta": meta(), "cases": []}
    if os.path.exists(path):
        res = json.load(open(path))
    done = {(c["k"], c["method"]) for c in res["cases"]}
    for k in (3, 4):
        re, im = problems.lu_matrix(n, k, 1, populate_lower=True, renorm=ref_renorm_planes)
        for meth in ("3m", "4m"):
            if (k, meth) in done:
                continue
            rec, f = _lu_record(re, im, K, meth)
            rec.update(seed=1, n=n, k=k, input_digest=digest(re, im))
            res["cases"].append(rec)
            print("cfg3", k, meth, rec["seconds"], flush=True)
            with open(path, "w") as fh:
                json.dump(res, fh)


def gen_ozaki():
    """ozaki.py: split parts/scales, rgemm_ozaki, cgemm and lu_blocked with
    real_kernel="ozaki" -- the f1 row's golden vectors."""
    from mpclu import ozaki_split, rgemm_ozaki

    rng = np.random.default_rng(20240802)
    out = {}

    def rmat(r, c, k):
        return mpclu.rmatrix.random_matrix(r, c, k, rng).data

    for k in (2, 3, 4):
        A = rmat(12, 10, k)
        B = rmat(10, 9, k)
        out[f"oz_A_k{k}"], out[f"oz_B_k{k}"] = A, B
        for d in (1, 3, 6):
            sa = ozaki_split(RealMatrix(A), d, "left")
            sb = ozaki_split(RealMatrix(B), d, "right")
            out[f"oz_sa_parts_k{k}_d{d}"] = np.array(sa.parts)
            out[f"oz_sa_scales_k{k}_d{d}"] = np.array(sa.scales)
            out[f"oz_sb_parts_k{k}_d{d}"] = np.array(sb.parts)
            out[f"oz_sb_scales_k{k}_d{d}"] = np.array(sb.scales)
        for d in ({2: (5, 6), 3: (7, 8), 4: (11, 12)}[k]):
            out[f"oz_C_k{k}_d{d}"] = rgemm_ozaki(RealMatrix(A), RealMatrix(B), d).data
        out[f"oz_C_k{k}_d4_sb12"] = rgemm_ozaki(RealMatrix(A), RealMatrix(B), 4, split_bits=12).data
        Ar, Ai, Br, Bi = rmat(13, 11, k), rmat(13, 11, k), rmat(11, 7, k), rmat(11, 7, k)
        out[f"ozc_Ar_k{k}"], out[f"ozc_Ai_k{k}"] = Ar, Ai
        out[f"ozc_Br_k{k}"], out[f"ozc_Bi_k{k}"] = Br, Bi
        for meth in ("3m", "4m"):
            C = cgemm(pc(Ar, Ai), pc(Br, Bi), KernelChoice(method=meth, real_kernel="ozaki"))
            out[f"ozc_{meth}_k{k}"] = np.array([C.re_plane.data, C.im_plane.data])
        n = 30
        re, im = rmat(n, n, k), rmat(n, n, k)
        re[0] -= 0.5
        out[f"ozlu_re_k{k}"], out[f"ozlu_im_k{k}"] = re, im
        for meth in ("3m", "4m"):
            f = lu_blocked(pc(re, im), 8, kc=KernelChoice(method=meth, real_kernel="ozaki"))
            out[f"ozlu_{meth}_k{k}"] = np.array([f.packed.re_plane.data, f.packed.im_plane.data])
            out[f"ozlu_{meth}_k{k}_piv"] = f.pivots
    path = os.path.join(GOLD, "ozaki.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    os.makedirs(GOLD, exist_ok=True)
    for what in sys.argv[1:]:
        if what == "cfg3small":
            gen_cfg3(n=512, K=128)
            continue
        {"small": gen_small, "cfg0": gen_cfg0, "cfg1": gen_cfg1, "cfg2": gen_cfg2,
         "cfg3": gen_cfg3, "ozaki": gen_ozaki, "cfg2_4m": gen_cfg2_4m,
         "ill": gen_ill}[what]()
