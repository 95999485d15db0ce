// Native local search of the online image placement (Alg. 1 line 8,
// PAPER.md:640-660, Appendix C.1): steepest-ascent
// pairwise swaps under the p-norm relaxed objective, the scheme of
// /root/reference/pkg/src/splatsched/placement.py:182-281, reproduced swap
// for swap.
//
// Every candidate swap (a < b, W[a] != W[b], triu order) gets its O(1) load
// deltas and its relaxed value; the first strictly best one is applied while
// it improves by more than 1e-12 relative.  To keep the decisions identical
// to the numpy restatement the floating-point semantics are numpy's:
//   * elementwise x ** p (arrays): the power kernel numpy's ufunc runs on
//     this CPU -- square / sqrt / copy for the exponents 2, 0.5, 1, else
//     with AVX512_SKX SVML's __svml_pow8 from numpy's own extension module
//     (its address is passed in), else libm pow;
//   * Python-float / numpy-scalar powers (the final ** (1 / p) of a norm):
//     libm pow;
//   * array sums: numpy's pairwise summation (8 accumulators from n >= 8);
//   * left-to-right elementwise expressions exactly as placement.py writes
//     them (this file is built with -ffp-contract=off: no fused multiply-add).
// Candidates are evaluated in parallel (OpenMP) with a deterministic
// (value, index) argmin, so the thread count never changes the result.
#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "../../../include/splat_host.h"

namespace {

typedef __m512d (*vpow8_fn)(__m512d, __m512d);

__attribute__((target("avx512f"))) void pow_avx512(vpow8_fn f, const double* x, double y, double* out, int64_t n) {
  const __m512d vy = _mm512_set1_pd(y);
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) _mm512_storeu_pd(out + i, f(_mm512_loadu_pd(x + i), vy));
  if (i < n) {
    const __mmask8 m = (__mmask8)((1u << (n - i)) - 1u);
    const __m512d r = f(_mm512_maskz_loadu_pd(m, x + i), vy);
    _mm512_mask_storeu_pd(out + i, m, r);
  }
}

struct ArrayPow {
  vpow8_fn v8;  // numpy's SIMD power kernel, or null: libm
  void operator()(const double* x, double y, double* out, int64_t n) const {
    // np.power's own fast paths for a scalar exponent
    if (y == 2.0) {
      for (int64_t i = 0; i < n; ++i) out[i] = x[i] * x[i];
    } else if (y == 0.5) {
      for (int64_t i = 0; i < n; ++i) out[i] = std::sqrt(x[i]);
    } else if (y == 1.0) {
      for (int64_t i = 0; i < n; ++i) out[i] = x[i];
    } else if (v8) {
      pow_avx512(v8, x, y, out, n);
    } else {
      for (int64_t i = 0; i < n; ++i) out[i] = std::pow(x[i], y);
    }
  }
};

// numpy pairwise_sum for a contiguous float64 array (n <= 128 here: N ranks)
double np_sum(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] += a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  const int64_t n2 = (n / 2) - ((n / 2) % 8);
  return np_sum(a, n2) + np_sum(a + n2, n - n2);
}

struct Search {
  int64_t B;
  int32_t N;
  double beta, gamma, delta, p;
  bool finite;
  ArrayPow apow;

  // _norm(x, p) = float(np.power(x, p).sum() ** (1 / p)); max for p = inf
  double norm(const std::vector<double>& x) const {
    if (!finite) {
      double m = -std::numeric_limits<double>::infinity();
      for (double v : x) m = std::max(m, v);
      return x.empty() ? 0.0 : m;
    }
    std::vector<double> t(x.size());
    apow(x.data(), p, t.data(), (int64_t)x.size());
    return std::pow(np_sum(t.data(), (int64_t)t.size()), 1.0 / p);
  }
  double relaxed(const std::vector<double>& s, const std::vector<double>& r, const std::vector<double>& c) const {
    return beta * norm(s) + gamma * norm(r) + delta * norm(c);
  }
};

}  // namespace

extern "C" int32_t bs_local_search(int64_t B, int32_t N, const int64_t* A, int64_t* W, double beta, double gamma,
                                   double delta, double p, int32_t max_sweeps, double wall_time,
                                   const void* simd_pow, int32_t n_threads, double* history, int64_t* n_history) {
  if (B < 1 || N < 1 || !A || !W || !history || !n_history || !(p >= 1.0)) return BS_HOST_ERR_PARAMETER;
  for (int64_t j = 0; j < B; ++j)
    if (W[j] < 0 || W[j] >= N) return BS_HOST_ERR_PARAMETER;
  const auto t_start = std::chrono::steady_clock::now();
  Search s{B, N, beta, gamma, delta, p, !std::isinf(p), ArrayPow{reinterpret_cast<vpow8_fn>(const_cast<void*>(simd_pow))}};
  // compute_loads (integer) then float64, as local_search does
  std::vector<int64_t> rowsum_i(B, 0), colsum(N, 0), own(N, 0), recv_i(N, 0), comp_i(N, 0);
  for (int64_t j = 0; j < B; ++j) {
    for (int k = 0; k < N; ++k) {
      rowsum_i[j] += A[j * N + k];
      colsum[k] += A[j * N + k];
    }
    const int64_t local = A[j * N + W[j]];
    own[W[j]] += local;
    recv_i[W[j]] += rowsum_i[j] - local;
    comp_i[W[j]] += rowsum_i[j];
  }
  std::vector<double> send(N), recv(N), comp(N), rows(B), Af(B * N);
  for (int k = 0; k < N; ++k) {
    send[k] = (double)(colsum[k] - own[k]);
    recv[k] = (double)recv_i[k];
    comp[k] = (double)comp_i[k];
  }
  for (int64_t j = 0; j < B; ++j) rows[j] = (double)rowsum_i[j];
  for (int64_t e = 0; e < B * N; ++e) Af[e] = (double)A[e];

  int64_t nh = 0;
  history[nh++] = s.relaxed(send, recv, comp);
  const int64_t n_pairs = B * (B - 1) / 2;
  std::vector<int32_t> pa, pb;  // live candidates in triu order
  pa.reserve(n_pairs);
  pb.reserve(n_pairs);
  const int nt = n_threads > 0 ? n_threads : 1;
  std::vector<double> sa(n_pairs), sb(n_pairs), ra(n_pairs), rb(n_pairs), ca(n_pairs), cb(n_pairs), val(n_pairs);
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (wall_time >= 0.0 &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count() > wall_time)
      break;
    pa.clear();
    pb.clear();
    for (int64_t a = 0; a < B; ++a)
      for (int64_t b = a + 1; b < B; ++b)
        if (W[a] != W[b]) {
          pa.push_back((int32_t)a);
          pb.push_back((int32_t)b);
        }
    const int64_t L = (int64_t)pa.size();
    if (L == 0) break;
    double ps[3] = {0.0, 0.0, 0.0};
    if (s.finite) {
      std::vector<double> t(N);
      s.apow(send.data(), p, t.data(), N);
      ps[0] = np_sum(t.data(), N);
      s.apow(recv.data(), p, t.data(), N);
      ps[1] = np_sum(t.data(), N);
      s.apow(comp.data(), p, t.data(), N);
      ps[2] = np_sum(t.data(), N);
    }
    // per-thread minimum over a contiguous block of candidates; the blocks
    // are combined in order, so ties resolve to the first (a, b) like argmin
    std::vector<double> best_v(nt, std::numeric_limits<double>::infinity());
    std::vector<int64_t> best_i(nt, -1);
    const double inv_p = 1.0 / p;
#pragma omp parallel num_threads(nt)
    {
      const int tid = omp_get_thread_num(), T = omp_get_num_threads();
      const int64_t lo = L * tid / T, hi = L * (tid + 1) / T;
      constexpr int64_t kBlk = 256;
      double x[6][kBlk], y[6][kBlk], nrm[3][kBlk];
      for (int64_t c0 = lo; c0 < hi; c0 += kBlk) {
        const int64_t n = std::min(kBlk, hi - c0);
        for (int64_t q = 0; q < n; ++q) {
          const int64_t c = c0 + q, a = pa[c], b = pb[c], ka = W[a], kb = W[b];
          sa[c] = send[ka] + Af[a * N + ka] - Af[b * N + ka];
          sb[c] = send[kb] + Af[b * N + kb] - Af[a * N + kb];
          ra[c] = recv[ka] + (rows[b] - Af[b * N + ka]) - (rows[a] - Af[a * N + ka]);
          rb[c] = recv[kb] + (rows[a] - Af[a * N + kb]) - (rows[b] - Af[b * N + kb]);
          ca[c] = comp[ka] + rows[b] - rows[a];
          cb[c] = comp[kb] + rows[a] - rows[b];
        }
        const std::vector<double>* vecs[3] = {&send, &recv, &comp};
        const double* na[3] = {sa.data() + c0, ra.data() + c0, ca.data() + c0};
        const double* nb[3] = {sb.data() + c0, rb.data() + c0, cb.data() + c0};
        for (int term = 0; term < 3; ++term) {
          const std::vector<double>& v = *vecs[term];
          if (s.finite) {
            // s = pow_sum - vec[ia]**p - vec[ib]**p + na**p + nb**p; max(s, 0) ** (1/p)
            for (int64_t q = 0; q < n; ++q) {
              x[0][q] = v[W[pa[c0 + q]]];
              x[1][q] = v[W[pb[c0 + q]]];
            }
            s.apow(x[0], p, y[0], n);
            s.apow(x[1], p, y[1], n);
            s.apow(na[term], p, y[2], n);
            s.apow(nb[term], p, y[3], n);
            for (int64_t q = 0; q < n; ++q) {
              const double t = ps[term] - y[0][q] - y[1][q] + y[2][q] + y[3][q];
              x[2][q] = std::max(t, 0.0);  // np.maximum(s, 0.0) (no NaN here)
            }
            s.apow(x[2], inv_p, nrm[term], n);
          } else {
            // max over the entries other than the two replaced (the top-3 rule)
            for (int64_t q = 0; q < n; ++q) {
              const int64_t ia = W[pa[c0 + q]], ib = W[pb[c0 + q]];
              double others = -std::numeric_limits<double>::infinity();
              for (int k = 0; k < N; ++k)
                if (k != ia && k != ib && v[k] > others) others = v[k];
              nrm[term][q] = std::max(std::max(na[term][q], nb[term][q]), others);
            }
          }
        }
        for (int64_t q = 0; q < n; ++q) {
          const double vq = beta * nrm[0][q] + gamma * nrm[1][q] + delta * nrm[2][q];
          val[c0 + q] = vq;
          if (vq < best_v[tid]) {
            best_v[tid] = vq;
            best_i[tid] = c0 + q;
          }
        }
      }
    }
    int64_t bi = -1;
    double bv = std::numeric_limits<double>::infinity();
    for (int t = 0; t < nt; ++t)
      if (best_i[t] >= 0 && (bi < 0 || best_v[t] < bv)) {
        bv = best_v[t];
        bi = best_i[t];
      }
    if (bi < 0) bi = 0;  // all values NaN/inf: argmin returns the first
    const double cur = history[nh - 1];
    if (val[bi] >= cur - 1e-12 * std::max(std::fabs(cur), 1.0)) break;
    const int64_t xa = pa[bi], yb = pb[bi], wx = W[xa], wy = W[yb];
    send[wx] = sa[bi];
    send[wy] = sb[bi];
    recv[wx] = ra[bi];
    recv[wy] = rb[bi];
    comp[wx] = ca[bi];
    comp[wy] = cb[bi];
    W[xa] = wy;
    W[yb] = wx;
    history[nh++] = s.relaxed(send, recv, comp);
  }
  *n_history = nh;
  return BS_HOST_OK;
}

// Elementwise power with the kernel bs_local_search would use (simd_pow or
// libm): lets the caller check it against numpy's np.power on this CPU.
extern "C" int32_t bs_array_pow(const double* x, double y, double* out, int64_t n, const void* simd_pow) {
  if (n < 0 || (n > 0 && (!x || !out))) return BS_HOST_ERR_PARAMETER;
  ArrayPow{reinterpret_cast<vpow8_fn>(const_cast<void*>(simd_pow))}(x, y, out, n);
  return BS_HOST_OK;
}
