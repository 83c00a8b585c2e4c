// expansion.cuh -- device multi-component (DD/TD/QD) expansion arithmetic.
//
// Bit-exact restatement of the reference's numba kernels
// (/root/reference/pkg/src/mpclu/_kernels.py, cited per function) for sm_100a.
// Rules that make the GPU bits equal the reference's:
//   * every FP64 operation is an explicit round-to-nearest intrinsic
//     (__dadd_rn/__dsub_rn/__dmul_rn), so nvcc can never contract a*b+c into
//     a DFMA (the reference runs without FMA contraction, _kernels.py:8-9);
//   * the only DFMA is TwoProd's error term, fma(a,b,-a*b), which equals the
//     reference's Dekker error term exactly for in-range operands;
//   * the k>=3 renormalization keeps the reference's data-dependent control
//     flow (sort by (|v| desc, v desc), VecSum, extraction with early break,
//     repeat-while-overlapping <= 6) using a sorting network and predication
//     instead of dynamic indexing so everything stays in registers.
// Comparisons that only steer control flow are done on the integer pipe
// (bit patterns) to keep the FP64 pipe for arithmetic.
#pragma once
#include <cstdint>

#include "sortnet.h"

namespace mpc {

constexpr int SORTNET_MAX = 41;  // largest SortNet in sortnet.h

#define MPC_DI __device__ __forceinline__

MPC_DI double dadd(double a, double b) { return __dadd_rn(a, b); }
MPC_DI double dsub(double a, double b) { return __dsub_rn(a, b); }
MPC_DI double dmul(double a, double b) { return __dmul_rn(a, b); }

MPC_DI uint64_t bits(double x) { return (uint64_t)__double_as_longlong(x); }
MPC_DI uint64_t absbits(double x) { return bits(x) & 0x7FFFFFFFFFFFFFFFull; }
// x != 0 (either sign); NaN counts as nonzero, like the bit test it replaces
// (one DSETP on the FP64 pipe instead of integer compare work)
MPC_DI bool is_nonzero(double x) { return x != 0.0; }

// ---------------------------------------------------------------- EFTs
// _kernels.py:28-34
MPC_DI void two_sum(double a, double b, double& s, double& e) {
  double ss = dadd(a, b);
  double bb = dsub(ss, a);
  e = dadd(dsub(a, dsub(ss, bb)), dsub(b, bb));
  s = ss;
}
// _kernels.py:37-42
MPC_DI void quick_two_sum(double a, double b, double& s, double& e) {
  double ss = dadd(a, b);
  e = dsub(b, dsub(ss, a));
  s = ss;
}
// _kernels.py:45-60 (Dekker there; FMA form here, bit-identical in range)
MPC_DI void two_prod(double a, double b, double& p, double& e) {
  double pp = dmul(a, b);
  e = __fma_rn(a, b, -pp);
  p = pp;
}

// ------------------------------------------------------- DD fast paths
// _kernels.py:146-155 (accurate add)
MPC_DI void dd_add(double x0, double x1, double y0, double y1, double& r0, double& r1) {
  double s1, s2, t1, t2;
  two_sum(x0, y0, s1, s2);
  two_sum(x1, y1, t1, t2);
  s2 = dadd(s2, t1);
  quick_two_sum(s1, s2, s1, s2);
  s2 = dadd(s2, t2);
  quick_two_sum(s1, s2, r0, r1);
}
// _kernels.py:158-164
MPC_DI void dd_mul(double x0, double x1, double y0, double y1, double& r0, double& r1) {
  double p, e;
  two_prod(x0, y0, p, e);
  double t = dadd(dmul(x0, y1), dmul(x1, y0));
  e = dadd(e, dadd(t, dmul(x1, y1)));
  quick_two_sum(p, e, r0, r1);
}

// ------------------------------------------------------------ expansion
template <int K>
struct Exp {
  double c[K];
};

template <int K>
MPC_DI Exp<K> exp_zero() {
  Exp<K> r;
#pragma unroll
  for (int i = 0; i < K; i++) r.c[i] = 0.0;
  return r;
}

template <int K>
MPC_DI Exp<K> exp_neg(const Exp<K>& x) {
  Exp<K> r;
#pragma unroll
  for (int i = 0; i < K; i++) r.c[i] = -x.c[i];
  return r;
}

// exp_abs_core, _kernels.py:258-265
template <int K>
MPC_DI Exp<K> exp_abs(const Exp<K>& x) {
  return (x.c[0] < 0.0) ? exp_neg(x) : x;
}

// Sort key for (|v| desc, v desc): (absbits << 1) | !sign -- a bijection on
// non-NaN doubles, so the network sorts the keys alone and the values are
// rebuilt from them afterwards (one 64-bit max / min pair per comparator).
// The order equals the reference's except among zeros (+0 now precedes -0,
// the reference treats them as equal): zeros always form the tail and their
// order cannot change the VecSum sweep (every TwoSum of two zeros gives the
// same sum and a +0 error in either order), so renorm's output is
// bit-identical.  Padding slots (i >= m) get key 0 (= -0): they sink to the
// end, and a padding key that ties with a real -0 rebuilds the same -0.
MPC_DI uint64_t sort_key(double v) {
  const uint64_t b = bits(v);
  return (b << 1) | ((b >> 63) ^ 1ull);
}
MPC_DI double from_key(uint64_t k) {
  return __longlong_as_double((long long)((k >> 1) | ((~k & 1ull) << 63)));
}

// _sort_desc, _kernels.py:67-78, on buf[0..m) (m <= M, runtime).  A sorting
// network (sortnet.h) replaces the insertion sort: the sorted sequence is
// the same except for the relative order of equal keys, i.e. identical
// values (no effect) -- see sort_key for the zeros.
template <int M>
MPC_DI void sort_desc(double (&buf)[M], int m) {
  uint64_t key[M];
  if constexpr (M > SORTNET_MAX) {
    // k = 8 verification kernels (exp_mul: 71 terms): the reference's own
    // insertion sort, on the keys in local memory (not unrolled)
    for (int i = 0; i < m; i++) {
      const uint64_t v = sort_key(buf[i]);
      int j = i - 1;
      while (j >= 0 && key[j] < v) {
        key[j + 1] = key[j];
        j--;
      }
      key[j + 1] = v;
    }
    for (int i = 0; i < M; i++) buf[i] = from_key(i < m ? key[i] : 0ull);
  } else {
#pragma unroll
    for (int i = 0; i < M; i++) key[i] = (i < m) ? sort_key(buf[i]) : 0ull;
    SortNet<M>::apply([&](int a, int b) {
      const uint64_t ka = key[a], kb = key[b];
      key[a] = ka > kb ? ka : kb;
      key[b] = ka > kb ? kb : ka;
    });
#pragma unroll
    for (int i = 0; i < M; i++) buf[i] = from_key(key[i]);
  }
}

// _vecsum_extract, _kernels.py:81-105, on buf[0..m) (m <= M runtime)
template <int M, int K>
MPC_DI void vecsum_extract(double (&buf)[M], int m, Exp<K>& out) {
  double s = 0.0;
  bool started = false;
#pragma unroll
  for (int i = M - 1; i >= 0; i--) {
    if (i < m) {
      if (!started) {
        s = buf[i];
        started = true;
      } else {
        double e;
        two_sum(buf[i], s, s, e);
        buf[i + 1 < M ? i + 1 : M - 1] = e;
      }
    }
  }
  buf[0] = s;
#pragma unroll
  for (int i = 0; i < K; i++) out.c[i] = 0.0;
  int j = 0;
  double eps = buf[0];
  bool done = false;
#pragma unroll
  for (int i = 0; i < M - 1; i++) {
    if (!done && i < m - 1) {
      double r, enew;
      two_sum(eps, buf[i + 1], r, enew);
      if (is_nonzero(enew)) {
        if (j >= K - 1) {
          eps = r;
          done = true;
        } else {
          // j <= K - 2 here, and j <= i: only those slots can take r
#pragma unroll
          for (int q = 0; q < K - 1; q++)
            if (q <= i && q == j) out.c[q] = r;
          j++;
          eps = enew;
        }
      } else {
        eps = r;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < K; q++)
    if (q == j) out.c[q] = eps;
}

// np.spacing(|x|) for the overlap test
MPC_DI double spacing_abs(double x) {
  uint64_t a = absbits(x);
  double ax = __longlong_as_double((long long)a);
  if (a >= 0x7FF0000000000000ull) return dsub(ax, ax);  // inf/nan -> nan
  double nx = __longlong_as_double((long long)(a + 1ull));
  return dsub(nx, ax);
}

// _is_nonoverlapping, _kernels.py:108-121
template <int K>
MPC_DI bool is_nonoverlapping(const Exp<K>& o) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < K - 1; i++) {
    double hi = o.c[i], lo = o.c[i + 1];
    if (!is_nonzero(hi)) {
      if (is_nonzero(lo)) ok = false;
    } else {
      double half = dmul(0.5, spacing_abs(hi));
      if (fabs(lo) > half || dadd(hi, lo) != hi) ok = false;
    }
  }
  return ok;
}

// the part of renorm after the sort (VecSum, extraction, repeat pass)
template <int M, int K>
MPC_DI Exp<K> renorm_sorted(double (&buf)[M]) {
  Exp<K> out;
  vecsum_extract<M, K>(buf, M, out);
  int it = 0;
  while (!is_nonoverlapping<K>(out) && it < 6) {
    double b2[K];
#pragma unroll
    for (int i = 0; i < K; i++) b2[i] = out.c[i];
    vecsum_extract<K, K>(b2, K, out);
    it++;
  }
  return out;
}

// Structured sort for renorm's term lists: the caller lays buf out as
// consecutive bands (compile-time sizes B...) that are each sorted by a small
// network (e.g. exp_mul's magnitude levels), or -- MERGE -- as two sorted
// runs merged by a merge network.  If the result is not fully sorted (bands
// overlap, zeros, unnormalized operands) the full network sorts it -- any
// permutation sorts to the same sequence, so the outcome is always exactly
// sort_desc's and renorm's bits do not change; the cheap path only has to
// be right for the common case.
template <int OFF, int N, typename F>
MPC_DI void net_at(F&& ce) {
  SortNet<N>::apply([&](int a, int b) { ce(a + OFF, b + OFF); });
}

// merge networks for two sorted runs of K (positions [0, K) and [K, 2K)),
// 0-1 verified over all pairs of sorted runs
template <int K>
struct MergeNet;
template <>
struct MergeNet<3> {
  template <typename F>
  MPC_DI static void apply(F&& ce) {
    ce(2, 3); ce(0, 2); ce(1, 2); ce(2, 4); ce(1, 5); ce(3, 5); ce(1, 2); ce(3, 4);
  }
};
template <>
struct MergeNet<4> {
  template <typename F>
  MPC_DI static void apply(F&& ce) {
    ce(0, 4); ce(2, 6); ce(2, 4); ce(1, 5); ce(3, 7); ce(3, 5); ce(1, 2); ce(3, 4); ce(5, 6);
  }
};

// exp_mul's magnitude bands for k = 3, 4 (see exp_mul): sizes per level
template <int K>
struct MulBands;
template <>
struct MulBands<3> {  // p00 | e00 p01 p10 | e01 e10 q02 q11 q20 | q12 q21
  template <typename F>
  MPC_DI static void apply(F&& ce) {
    net_at<1, 3>(ce);
    net_at<4, 5>(ce);
    net_at<9, 2>(ce);
  }
};
template <>
struct MulBands<4> {  // p00 | e00 p01 p10 | e01 e10 p02 p11 p20 | e02 e11 e20 q03 q12 q21 q30 | q13 q22 q31
  template <typename F>
  MPC_DI static void apply(F&& ce) {
    net_at<1, 3>(ce);
    net_at<4, 5>(ce);
    net_at<9, 7>(ce);
    net_at<16, 3>(ce);
  }
};

// exp_div's residual update terms by level (see exp_div): bands of 2, then
// 3 per lower level, then the last TwoProd error alone
template <int K>
struct DivBands {
  template <typename F>
  MPC_DI static void apply(F&& ce) {
    net_at<0, 2>(ce);
    if constexpr (K >= 2) net_at<2, 3>(ce);
    if constexpr (K >= 3) net_at<5, 3>(ce);
    if constexpr (K >= 4) net_at<8, 3>(ce);
  }
};

// a strictly precedes b in _sort_desc's order (|v| desc, then v desc),
// compared on the FP64 pipe (DSETP with |.| operand modifiers); zeros of
// either sign compare equal, as in the reference's insertion sort
MPC_DI bool precedes(double a, double b) {
  const double fa = fabs(a), fb = fabs(b);
  return fa > fb || (fa == fb && a > b);
}

// Structured sort of a full term list (every slot a real term): the
// caller's presort network runs with a magnitude-only comparator (one DSETP
// + the selects of the swap), the result is checked pair by pair in the
// exact order, and only an unsorted result (bands overlap, or two terms of
// equal magnitude and opposite sign) runs the exact full network.  Any
// permutation sorts to the same sequence up to the order of zeros, which
// cannot change the VecSum sweep (see sort_key), so renorm's bits do not
// depend on which path ran.  Doubles are compared directly: no key
// construction / reconstruction (the integer compare-and-select of the key
// network was the issue bottleneck of the TD / QD kernels, ncu r2).
template <int M, typename Pre>
MPC_DI void sort_desc_pre(double (&buf)[M], Pre&& pre) {
  auto ce_abs = [&](int a, int b) {
    const double va = buf[a], vb = buf[b];
    const bool sw = fabs(vb) > fabs(va);
    buf[a] = sw ? vb : va;
    buf[b] = sw ? va : vb;
  };
  pre(ce_abs);
  bool bad = false;
#pragma unroll
  for (int i = 0; i + 1 < M; i++) bad |= precedes(buf[i + 1], buf[i]);
  if (bad) {
    SortNet<M>::apply([&](int a, int b) {
      const double va = buf[a], vb = buf[b];
      const bool sw = precedes(vb, va);
      buf[a] = sw ? vb : va;
      buf[b] = sw ? va : vb;
    });
  }
}

// renorm, _kernels.py:124-139 on buf[0..m) (buf clobbered)
template <int M, int K>
MPC_DI Exp<K> renorm(double (&buf)[M], int m) {
  Exp<K> out;
  sort_desc<M>(buf, m);
  vecsum_extract<M, K>(buf, m, out);
  int it = 0;
  while (!is_nonoverlapping<K>(out) && it < 6) {
    double b2[K];
#pragma unroll
    for (int i = 0; i < K; i++) b2[i] = out.c[i];
    vecsum_extract<K, K>(b2, K, out);
    it++;
  }
  return out;
}

// exp_add_core, _kernels.py:174-184
template <int K>
MPC_DI Exp<K> exp_add(const Exp<K>& x, const Exp<K>& y) {
  if constexpr (K == 2) {
    Exp<2> r;
    dd_add(x.c[0], x.c[1], y.c[0], y.c[1], r.c[0], r.c[1]);
    return r;
  } else {
    double buf[2 * K];
#pragma unroll
    for (int i = 0; i < K; i++) {
      buf[i] = x.c[i];
      buf[K + i] = y.c[i];
    }
    // normalized operands are sorted runs: merge, verify, else full sort
    // (k > 4: the verification kernels only, plain renorm)
    if constexpr (K <= 4) {
      sort_desc_pre<2 * K>(buf, [](auto&& ce) { MergeNet<K>::apply(ce); });
      return renorm_sorted<2 * K, K>(buf);
    } else {
      return renorm<2 * K, K>(buf, 2 * K);
    }
  }
}

// exp_sub_core, _kernels.py:187-197
template <int K>
MPC_DI Exp<K> exp_sub(const Exp<K>& x, const Exp<K>& y) {
  if constexpr (K == 2) {
    Exp<2> r;
    dd_add(x.c[0], x.c[1], -y.c[0], -y.c[1], r.c[0], r.c[1]);
    return r;
  } else {
    double buf[2 * K];
#pragma unroll
    for (int i = 0; i < K; i++) {
      buf[i] = x.c[i];
      buf[K + i] = -y.c[i];
    }
    if constexpr (K <= 4) {
      sort_desc_pre<2 * K>(buf, [](auto&& ce) { MergeNet<K>::apply(ce); });
      return renorm_sorted<2 * K, K>(buf);
    } else {
      return renorm<2 * K, K>(buf, 2 * K);
    }
  }
}

// exp_mul_core, _kernels.py:200-222
template <int K>
MPC_DI Exp<K> exp_mul(const Exp<K>& x, const Exp<K>& y) {
  if constexpr (K == 2) {
    Exp<2> r;
    dd_mul(x.c[0], x.c[1], y.c[0], y.c[1], r.c[0], r.c[1]);
    return r;
  } else {
    // the reference's term list (_kernels.py:205-219): TwoProd pairs of
    // levels 0..k-2, plain products of levels k-1 and k.  The order of the
    // list does not matter to renorm (it sorts), so it is laid out by
    // magnitude level -- p00 | e00 p01 p10 | ... -- for the banded presort.
    constexpr int M = K * K + K - 1;
    double p[K - 1][K - 1], e[K - 1][K - 1];
#pragma unroll
    for (int s = 0; s < K - 1; s++)
#pragma unroll
      for (int i = 0; i < s + 1; i++) two_prod(x.c[i], y.c[s - i], p[s][i], e[s][i]);
    double buf[M];
    int m = 0;
    buf[m++] = p[0][0];
#pragma unroll
    for (int L = 1; L <= K; L++) {
      if (L - 1 <= K - 2) {
#pragma unroll
        for (int i = 0; i < L; i++) buf[m++] = e[L - 1][i];
      }
      if (L <= K - 2) {
#pragma unroll
        for (int i = 0; i < L + 1; i++) buf[m++] = p[L][i];
      }
      if (L == K - 1) {
#pragma unroll
        for (int i = 0; i < K; i++) buf[m++] = dmul(x.c[i], y.c[K - 1 - i]);
      }
      if (L == K) {
#pragma unroll
        for (int i = 1; i < K; i++) buf[m++] = dmul(x.c[i], y.c[K - i]);
      }
    }
    if constexpr (K <= 4) {
      sort_desc_pre<M>(buf, [](auto&& ce) { MulBands<K>::apply(ce); });
      return renorm_sorted<M, K>(buf);
    } else {
      return renorm<M, K>(buf, M);
    }
  }
}

// exp_div_core, _kernels.py:225-255 (long division, k+1 quotient digits;
// generic renorm even for k = 2, exactly as the reference)
template <int K>
MPC_DI Exp<K> exp_div(const Exp<K>& x, const Exp<K>& y) {
  double q[K + 1];
#pragma unroll
  for (int i = 0; i < K + 1; i++) q[i] = 0.0;
  Exp<K> r = x;
  int nq = 0;
  bool stop = false;
#pragma unroll
  for (int it = 0; it < K + 1; it++) {
    if (!stop) {
      double qi = __ddiv_rn(r.c[0], y.c[0]);
#pragma unroll
      for (int s = 0; s < K + 1; s++)
        if (s == it) q[s] = qi;
      nq++;
      if (!is_nonzero(qi) || it == K) {
        stop = true;
      } else {
        // the term list r, -p_i, -e_i (i < k) laid out by magnitude level
        // -- r0 -p0 | r1 -e0 -p1 | ... | -e_{k-1} -- for the banded presort
        // (renorm sorts, so the list order is free; same bits)
        double p[K], e[K];
#pragma unroll
        for (int i = 0; i < K; i++) two_prod(qi, y.c[i], p[i], e[i]);
        double buf[3 * K];
        int m = 0;
        buf[m++] = r.c[0];
        buf[m++] = -p[0];
#pragma unroll
        for (int L = 1; L < K; L++) {
          buf[m++] = r.c[L];
          buf[m++] = -e[L - 1];
          buf[m++] = -p[L];
        }
        buf[m++] = -e[K - 1];
        if constexpr (K <= 4) {
          sort_desc_pre<3 * K>(buf, [](auto&& ce) { DivBands<K>::apply(ce); });
          r = renorm_sorted<3 * K, K>(buf);
        } else {
          r = renorm<3 * K, K>(buf, 3 * K);
        }
      }
    }
  }
  return renorm<K + 1, K>(q, nq);
}

// ------------------------------------------------------ complex scalars
template <int K>
struct Cx {
  Exp<K> re, im;
};

// cmul_3m_core, _kernels.py:527-537
template <int K>
MPC_DI Cx<K> cmul3(const Exp<K>& ar, const Exp<K>& ai, const Exp<K>& br, const Exp<K>& bi) {
  Exp<K> s1 = exp_mul(ar, br);
  Exp<K> s2 = exp_mul(ai, bi);
  Cx<K> o;
  o.re = exp_sub(s1, s2);
  Exp<K> s3 = exp_add(ar, ai);
  Exp<K> t = exp_add(br, bi);
  s3 = exp_mul(s3, t);
  s3 = exp_sub(s3, s1);
  o.im = exp_sub(s3, s2);
  return o;
}

// cmul_3m_core with the two operand sums precomputed (same bits: the sums are
// the same exp_add calls, hoisted out of the inner loop)
template <int K>
MPC_DI Cx<K> cmul3_pre(const Exp<K>& ar, const Exp<K>& ai, const Exp<K>& sa, const Exp<K>& br,
                       const Exp<K>& bi, const Exp<K>& sb) {
  Exp<K> s1 = exp_mul(ar, br);
  Exp<K> s2 = exp_mul(ai, bi);
  Cx<K> o;
  o.re = exp_sub(s1, s2);
  Exp<K> s3 = exp_mul(sa, sb);
  s3 = exp_sub(s3, s1);
  o.im = exp_sub(s3, s2);
  return o;
}

// cmul_4m_core, _kernels.py:539-546
template <int K>
MPC_DI Cx<K> cmul4(const Exp<K>& ar, const Exp<K>& ai, const Exp<K>& br, const Exp<K>& bi) {
  Exp<K> s1 = exp_mul(ar, br);
  Exp<K> s2 = exp_mul(ai, bi);
  Cx<K> o;
  o.re = exp_sub(s1, s2);
  s1 = exp_mul(ai, br);
  s2 = exp_mul(ar, bi);
  o.im = exp_add(s1, s2);
  return o;
}

template <int K>
MPC_DI Cx<K> cmul(bool use3m, const Exp<K>& ar, const Exp<K>& ai, const Exp<K>& br,
                  const Exp<K>& bi) {
  return use3m ? cmul3(ar, ai, br, bi) : cmul4(ar, ai, br, bi);
}

// cdiv_core, _kernels.py:549-561
template <int K>
MPC_DI Cx<K> cdiv(const Exp<K>& ar, const Exp<K>& ai, const Exp<K>& br, const Exp<K>& bi) {
  Exp<K> s1 = exp_mul(br, br);
  Exp<K> s2 = exp_mul(bi, bi);
  s1 = exp_add(s1, s2);  // d
  s2 = exp_mul(ar, br);
  Exp<K> s3 = exp_mul(ai, bi);
  s2 = exp_add(s2, s3);
  s3 = exp_mul(ai, br);
  Exp<K> t = exp_mul(ar, bi);
  s3 = exp_sub(s3, t);
  Cx<K> o;
  o.re = exp_div(s2, s1);
  o.im = exp_div(s3, s1);
  return o;
}

// pivot comparator, _pivot_row's test (cand - best)[0] > 0 (_kernels.py:586-587)
template <int K>
MPC_DI bool exp_greater(const Exp<K>& a, const Exp<K>& b) {
  Exp<K> d = exp_sub(a, b);
  return d.c[0] > 0.0;
}

}  // namespace mpc
