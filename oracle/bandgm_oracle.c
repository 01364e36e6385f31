/*
 * CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's banded operator loops
 * (/root/reference/proj, "bandgm").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product path (paper_1902_10078_b200/) never does.
 *
 * Parity pin: every function follows the reference loop nest, loop order and
 * division placement exactly, so with -ffp-contract=off it reproduces the
 * reference bit for bit.  tests/test_oracle.py checks that against the
 * reference sources compiled verbatim (oracle/_ref, built by oracle/Makefile)
 * and against the committed golden vectors in tests/golden/.
 *
 * Storage: a band with `lo` sub- and `up` super-diagonals of an n x n matrix
 * is a column-major (lo+up+1) x n array; entry (i, j) sits at storage row
 * i - j + up of column j (banded.hpp:1-11).  Batched entry points take
 * `batch` such arrays back to back and loop over matrices with OpenMP.
 *
 * Status codes (match paper_1902_10078_b200 / include/bandgm_b200.h):
 *   0 ok, 1 NotPositiveDefinite, 2 SingularDiagonal, 3 NonPositiveDiagonal,
 *   4 DimensionMismatch; `row` receives the failing row (errors.hpp:27-50).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_NOT_PD 1
#define ORC_SINGULAR 2
#define ORC_NONPOS 3
#define ORC_DIM 4

static const double kPivotFloor = 1e-300; /* kernels.hpp:20 */

typedef int64_t ix;

typedef struct {
  ix n, lo, up;
  double* d;
} band;

static inline ix imax(ix a, ix b) { return a > b ? a : b; }
static inline ix imin(ix a, ix b) { return a < b ? a : b; }
static inline ix rows_of(const band* a) { return a->lo + a->up + 1; }
/* unchecked in-band accessor, banded.hpp:64-65 */
static inline double* at(const band* a, ix i, ix j) {
  return &a->d[(i - j + a->up) + j * rows_of(a)];
}
static inline int in_band(const band* a, ix i, ix j) {
  const ix d = i - j;
  return i >= 0 && i < a->n && j >= 0 && j < a->n && d >= -a->up && d <= a->lo;
}
/* banded.hpp:69-71 */
static inline double at_or_zero(const band* a, ix i, ix j) {
  return in_band(a, i, j) ? *at(a, i, j) : 0.0;
}
/* symmetric mirrored read on a lower store, banded.hpp:129 */
static inline double sym(const band* s, ix i, ix j) { return i >= j ? *at(s, i, j) : *at(s, j, i); }

static band mk(ix n, ix lo, ix up, double* d) {
  band b = {n, lo, up, d};
  return b;
}
static double* zalloc(ix count) { return (double*)calloc((size_t)(count > 0 ? count : 1), sizeof(double)); }
static band alloc_band(ix n, ix lo, ix up) { return mk(n, lo, up, zalloc(n * (lo + up + 1))); }

/* ---------------------------------------------------------------- forward */

/* kernels_serial.cpp:12-32 (PAPER Alg. 1) */
static int chol1(ix n, ix bw, const double* qd, double* ld, ix* row) {
  band q = mk(n, bw, 0, (double*)qd), l = mk(n, bw, 0, ld);
  memset(ld, 0, sizeof(double) * (size_t)(n * (bw + 1)));
  for (ix i = 0; i < n; ++i) {
    const ix j0 = imax(0, i - bw);
    for (ix j = j0; j <= i; ++j) {
      double s = 0.0;
      for (ix m = j0; m < j; ++m) s += *at(&l, i, m) * *at(&l, j, m);
      if (i == j) {
        const double piv = *at(&q, i, i) - s;
        if (!(piv > kPivotFloor)) {
          *row = i;
          return ORC_NOT_PD;
        }
        *at(&l, i, i) = sqrt(piv);
      } else {
        *at(&l, i, j) = (*at(&q, i, j) - s) / *at(&l, j, j);
      }
    }
  }
  return ORC_OK;
}

/* kernels_serial.cpp:34-60 */
static int solve_vec1(ix n, ix bw, const double* ld, const double* v, int tr, double* x, ix* row) {
  band l = mk(n, bw, 0, (double*)ld);
  if (!tr) {
    for (ix i = 0; i < n; ++i) {
      double s = 0.0;
      for (ix k = imax(0, i - bw); k < i; ++k) s += *at(&l, i, k) * x[k];
      const double piv = *at(&l, i, i);
      if (fabs(piv) < kPivotFloor) {
        *row = i;
        return ORC_SINGULAR;
      }
      x[i] = (v[i] - s) / piv;
    }
  } else {
    for (ix i = n - 1; i >= 0; --i) {
      double s = 0.0;
      const ix k1 = imin(n - 1, i + bw);
      for (ix k = i + 1; k <= k1; ++k) s += *at(&l, k, i) * x[k];
      const double piv = *at(&l, i, i);
      if (fabs(piv) < kPivotFloor) {
        *row = i;
        return ORC_SINGULAR;
      }
      x[i] = (v[i] - s) / piv;
    }
  }
  return ORC_OK;
}

/* kernels_detail.hpp:58-72 */
static int solve_mat_entry(const band* l, const band* r, band* out, ix i, ix j, int tr, ix* row) {
  const ix n = l->n;
  const double piv = *at(l, i, i);
  if (fabs(piv) < 1e-300) {
    *row = i;
    return ORC_SINGULAR;
  }
  double s = 0.0;
  if (!tr) {
    for (ix m = imax(0, i - l->lo); m < i; ++m) s += *at(l, i, m) * at_or_zero(out, m, j);
  } else {
    const ix m1 = imin(n - 1, i + l->lo);
    for (ix m = i + 1; m <= m1; ++m) s += *at(l, m, i) * at_or_zero(out, m, j);
  }
  *at(out, i, j) = (at_or_zero(r, i, j) - s) / piv;
  return ORC_OK;
}

/* kernels_serial.cpp:62-78 (PAPER Alg. 4); out bands already clipped to n-1 */
static int solve_mat1(const band* l, const band* r, band* out, int tr, ix* row) {
  const ix n = l->n;
  memset(out->d, 0, sizeof(double) * (size_t)(n * rows_of(out)));
  if (!tr) {
    for (ix k = -out->up; k <= out->lo; ++k)
      for (ix i = imax(0, k); i <= imin(n - 1, n - 1 + k); ++i) {
        int st = solve_mat_entry(l, r, out, i, i - k, 0, row);
        if (st) return st;
      }
  } else {
    for (ix k = out->lo; k >= -out->up; --k)
      for (ix i = imax(0, k); i <= imin(n - 1, n - 1 + k); ++i) {
        int st = solve_mat_entry(l, r, out, i, i - k, 1, row);
        if (st) return st;
      }
  }
  return ORC_OK;
}

/* kernels_serial.cpp:80-104 (PAPER Alg. 3, Takahashi) */
static int subset1(ix n, ix bw, const double* ld, double* sd, ix* row) {
  band l = mk(n, bw, 0, (double*)ld), s = mk(n, bw, 0, sd);
  memset(sd, 0, sizeof(double) * (size_t)(n * (bw + 1)));
  double* vec = zalloc(n);
  for (ix i = 0; i < n; ++i) {
    vec[i] = *at(&l, i, i);
    if (fabs(vec[i]) < kPivotFloor) {
      free(vec);
      *row = i;
      return ORC_SINGULAR;
    }
  }
  for (ix j = n - 1; j >= 0; --j) {
    for (ix i = j; i >= imax(0, j - bw); --i) {
      double acc = 0.0;
      const ix m1 = imin(n - 1, i + bw);
      for (ix m = i + 1; m <= m1; ++m) acc += (*at(&l, m, i) / vec[i]) * sym(&s, m, j);
      double val = -acc;
      if (i == j) val += 1.0 / (vec[i] * vec[i]);
      *at(&s, j, i) = val;
    }
  }
  free(vec);
  return ORC_OK;
}

/* kernels_detail.hpp:16-28, one output column of a restricted product */
static void product_column(const band* a, const band* b, band* out, ix j) {
  const ix n = a->n;
  const ix i0 = imax(0, j - out->up), i1 = imin(n - 1, j + out->lo);
  for (ix i = i0; i <= i1; ++i) {
    const ix k0 = imax(imax(0, i - a->lo), j - b->up);
    const ix k1 = imin(imin(n - 1, i + a->up), j + b->lo);
    double s = 0.0;
    for (ix k = k0; k <= k1; ++k) s += *at(a, i, k) * *at(b, k, j);
    *at(out, i, j) = s;
  }
}
/* kernels_serial.cpp:106-113; `out` carries the clipped (ol, ou) */
static void product1(const band* a, const band* b, band* out) {
  memset(out->d, 0, sizeof(double) * (size_t)(out->n * rows_of(out)));
  for (ix j = 0; j < a->n; ++j) product_column(a, b, out, j);
}

/* kernels_detail.hpp:31-45 */
static void band_vec1(const band* b, const double* v, int tr, double* y) {
  const ix n = b->n;
  for (ix i = 0; i < n; ++i) {
    double s = 0.0;
    if (!tr) {
      const ix j0 = imax(0, i - b->lo), j1 = imin(n - 1, i + b->up);
      for (ix j = j0; j <= j1; ++j) s += *at(b, i, j) * v[j];
    } else {
      const ix j0 = imax(0, i - b->up), j1 = imin(n - 1, i + b->lo);
      for (ix j = j0; j <= j1; ++j) s += *at(b, j, i) * v[j];
    }
    y[i] = s;
  }
}

/* kernels_detail.hpp:48-54 and kernels_serial.cpp:124-131 */
static void outer1(const double* m, const double* v, band* out) {
  const ix n = out->n;
  memset(out->d, 0, sizeof(double) * (size_t)(n * rows_of(out)));
  for (ix j = 0; j < n; ++j) {
    const ix i0 = imax(0, j - out->up), i1 = imin(n - 1, j + out->lo);
    for (ix i = i0; i <= i1; ++i) *at(out, i, j) = m[i] * v[j];
  }
}

/* kernels.cpp:121-129 */
static int log_det1(ix n, ix bw, const double* ld, double* out, ix* row) {
  band l = mk(n, bw, 0, (double*)ld);
  double s = 0.0;
  for (ix i = 0; i < n; ++i) {
    const double d = *at(&l, i, i);
    if (!(d > 0.0)) {
      *row = i;
      return ORC_NONPOS;
    }
    s += log(d);
  }
  *out = s;
  return ORC_OK;
}

/* banded.cpp:159-167 */
static band transpose1(const band* a) {
  band t = alloc_band(a->n, a->up, a->lo);
  for (ix j = 0; j < a->n; ++j) {
    const ix i0 = imax(0, j - a->up), i1 = imin(a->n - 1, j + a->lo);
    for (ix i = i0; i <= i1; ++i) *at(&t, j, i) = *at(a, i, j);
  }
  return t;
}

/* ---------------------------------------------------------------- reverse */

/* grad.cpp:11-36 (PAPER Alg. 2); lb is consumed (overwritten) */
static void vjp_chol1(ix n, ix bw, const double* ld, double* lbd, double* qbd) {
  band l = mk(n, bw, 0, (double*)ld), lb = mk(n, bw, 0, lbd), qb = mk(n, bw, 0, qbd);
  memset(qbd, 0, sizeof(double) * (size_t)(n * (bw + 1)));
  for (ix i = n - 1; i >= 0; --i) {
    const ix j_stop = imax(0, i - bw);
    for (ix j = i; j >= j_stop; --j) {
      if (j == i) {
        *at(&qb, i, i) = 0.5 * *at(&lb, i, i) / *at(&l, i, i);
      } else {
        *at(&qb, i, j) = *at(&lb, i, j) / *at(&l, j, j);
        *at(&lb, j, j) -= *at(&lb, i, j) * *at(&l, i, j) / *at(&l, j, j);
      }
      const double q = *at(&qb, i, j);
      for (ix k = j - 1; k >= j_stop; --k) {
        *at(&lb, i, k) -= q * *at(&l, j, k);
        *at(&lb, j, k) -= q * *at(&l, i, k);
      }
    }
  }
}

/* grad.cpp:38-49 */
static int vjp_solve_vec1(ix n, ix bw, const double* ld, const double* s, const double* sb, int tr,
                          double* lbd, double* vb, ix* row) {
  int st = solve_vec1(n, bw, ld, sb, !tr, vb, row);
  if (st) return st;
  band lbar = mk(n, bw, 0, lbd);
  outer1(tr ? s : vb, tr ? vb : s, &lbar);
  for (ix c = 0; c < n * (bw + 1); ++c) lbd[c] *= -1.0;
  return ORC_OK;
}

/* grad.cpp:84-143 (PAPER Alg. 5) */
static int vjp_subset1(ix n, ix bw, const double* ld, const double* sd, const double* sbd,
                       double* lbd, ix* row) {
  band l = mk(n, bw, 0, (double*)ld), s = mk(n, bw, 0, (double*)sd);
  const ix r_bu = 2 * bw + 1, r_inv = 3 * bw + 2, r_bvec = r_inv + 1, wr = r_bvec + 1;
  double* ws = zalloc(wr * n);
#define WS(r, c) ws[(r) + (c) * wr]
  for (ix c = 0; c < n; ++c)
    for (ix r = 0; r <= bw; ++r) WS(bw + r, c) = sbd[r + c * (bw + 1)];
  for (ix i = 0; i < n; ++i) {
    const double piv = *at(&l, i, i);
    if (fabs(piv) < kPivotFloor) {
      free(ws);
      *row = i;
      return ORC_SINGULAR;
    }
    WS(r_inv, i) = 1.0 / piv;
  }
#define BS(i, j) WS((i) - (j) + bw, (j))
#define BU(i, m) WS(r_bu + (i) - (m) + bw, (m))
  for (ix j = 0; j < n; ++j) {
    for (ix i = imax(0, j - bw); i <= j; ++i) {
      if (i == j) WS(r_bvec, i) = BS(i, i);
      const double tmp = BS(j, i);
      BS(j, i) = 0.0;
      BS(i, j) += tmp;
      const double cur = BS(i, j);
      const double scale = cur * WS(r_inv, i);
      const ix m1 = imin(n - 1, i + bw);
      for (ix m = i + 1; m <= m1; ++m) {
        BU(i, m) -= sym(&s, m, j) * cur;
        BS(m, j) -= *at(&l, m, i) * scale;
      }
      BS(i, j) = 0.0;
    }
  }
  band lbar = mk(n, bw, 0, lbd);
  memset(lbd, 0, sizeof(double) * (size_t)(n * (bw + 1)));
  for (ix c = 0; c < n; ++c) {
    const double iv = WS(r_inv, c);
    const ix r1 = imin(n - 1, c + bw);
    double diag_sum = 0.0;
    for (ix r = c + 1; r <= r1; ++r) {
      *at(&lbar, r, c) = BU(c, r) * iv;
      diag_sum += BU(c, r) * *at(&l, r, c);
    }
    *at(&lbar, c, c) = (-2.0 * WS(r_bvec, c) * iv - diag_sum) * (iv * iv);
  }
#undef BU
#undef BS
#undef WS
  free(ws);
  return ORC_OK;
}

/* grad.cpp:145-151 (PAPER Table 1, band-band product) */
static void vjp_product1(const band* a, const band* b, const band* pb, band* ab, band* bb) {
  const ix n = a->n;
  band bt = transpose1(b), at_ = transpose1(a);
  /* product_band_band_restricted clips the requested band at n-1 (kernels.cpp:80-81) */
  product1(pb, &bt, ab);
  product1(&at_, pb, bb);
  (void)n;
  free(bt.d);
  free(at_.d);
}

/* grad.cpp:51-82 */
static int vjp_solve_mat1(const band* l, const band* s, const band* sb, ix rl, ix ru, int tr,
                          band* lb, band* rb, ix* row) {
  const ix n = l->n;
  int st;
  band t;
  if (!tr) {
    t = alloc_band(n, imin(sb->lo, n - 1), imin(imax(sb->up, ru), n - 1));
    st = solve_mat1(l, sb, &t, 1, row);
  } else {
    t = alloc_band(n, imin(imax(sb->lo, rl), n - 1), imin(sb->up, n - 1));
    st = solve_mat1(l, sb, &t, 0, row);
  }
  if (st) {
    free(t.d);
    return st;
  }
  memset(rb->d, 0, sizeof(double) * (size_t)(n * rows_of(rb)));
  for (ix j = 0; j < n; ++j) {
    const ix i0 = imax(0, j - rb->up), i1 = imin(n - 1, j + rb->lo);
    for (ix i = i0; i <= i1; ++i) *at(rb, i, j) = at_or_zero(&t, i, j);
  }
  if (!tr) {
    band st_ = transpose1(s);
    product1(&t, &st_, lb);
    free(st_.d);
  } else {
    band tt = transpose1(&t);
    product1(s, &tt, lb);
    free(tt.d);
  }
  for (ix c = 0; c < n * rows_of(lb); ++c) lb->d[c] *= -1.0;
  free(t.d);
  return ORC_OK;
}

/* grad.cpp:172-176 */
static void vjp_log_det1(ix n, ix bw, const double* ld, double cbar, double* lbd) {
  band l = mk(n, bw, 0, (double*)ld), lb = mk(n, bw, 0, lbd);
  memset(lbd, 0, sizeof(double) * (size_t)(n * (bw + 1)));
  for (ix i = 0; i < n; ++i) *at(&lb, i, i) = cbar / *at(&l, i, i);
}

/* ------------------------------------------------- config-3 composite
 * Restates infer::marginal_likelihood_partial (inference.cpp:140-163) with
 * every node observed, the precision Q = band(L L^T) built as in
 * precision_from_factor (inference.cpp:23-26), and the backward pass in the
 * exact node order Tape::backward would replay it (tape.cpp:435-451), then
 * chains Q_bar to L through grad::vjp_product_band_band(L, L^T, G)
 * (grad.cpp:145-151): L_bar = a_bar + transpose(b_bar).
 */
static const double kLog2Pi = 1.8378770664093454836; /* inference.cpp:15 */

static int mlik1(ix n, ix bw, const double* L, const double* y, double tau2, double* loss,
                 double* lbar_out, double* tau2_bar, ix* row) {
  const ix w = bw + 1;
  int st = ORC_OK;
  band Lb = mk(n, bw, 0, (double*)L);
  band Lt = transpose1(&Lb);
  band Q = alloc_band(n, bw, 0);
  product1(&Lb, &Lt, &Q); /* restricted(L, L^T, bw, 0) */
  const double nn = (double)n;
  /* forward, node by node */
  const double inv_tau = 1.0 / tau2;                   /* div */
  band A = alloc_band(n, bw, 0);                       /* add_diagonal_sym */
  memcpy(A.d, Q.d, sizeof(double) * (size_t)(n * w));
  for (ix i = 0; i < n; ++i) *at(&A, i, i) += 1.0 * inv_tau; /* scale_vec(mask=1) */
  double* Lp = zalloc(n * w);
  double* LQ = zalloc(n * w);
  double* wv = zalloc(n);
  double ldp = 0, ldq = 0;
  st = chol1(n, bw, A.d, Lp, row);
  if (st) goto done;
  st = solve_vec1(n, bw, Lp, y, 0, wv, row);
  if (st) goto done;
  st = log_det1(n, bw, Lp, &ldp, row);
  if (st) goto done;
  st = chol1(n, bw, Q.d, LQ, row);
  if (st) goto done;
  st = log_det1(n, bw, LQ, &ldq, row);
  if (st) goto done;
  {
    double yy = 0.0, ww = 0.0;
    for (ix i = 0; i < n; ++i) yy += y[i] * y[i];
    for (ix i = 0; i < n; ++i) ww += wv[i] * wv[i];
    double obj = -0.5 * nn * kLog2Pi;
    obj = obj + (-ldp);
    obj = obj + ldq;
    obj = obj + (-0.5 * nn) * log(tau2);
    obj = obj + (-0.5 * yy) * inv_tau;
    obj = obj + 0.5 * (ww * (inv_tau * inv_tau));
    *loss = obj;

    /* backward (node numbering in the comments follows creation order) */
    double g_inv = 0.0, g_tau2 = 0.0;
    const double g27 = 1.0 * 0.5;                 /* mul(0.5, .) */
    const double g25 = g27 * (inv_tau * inv_tau); /* mul(dot, inv^2) */
    const double g26 = g27 * ww;
    g_inv += g26 * inv_tau;                       /* mul(inv, inv): both operands */
    g_inv += g26 * inv_tau;
    double* gw = zalloc(n);                       /* dot(w, w): both operands */
    for (ix i = 0; i < n; ++i) gw[i] += g25 * wv[i];
    for (ix i = 0; i < n; ++i) gw[i] += g25 * wv[i];
    g_inv += 1.0 * (-0.5 * yy);                   /* mul(-0.5 yy, inv) */
    const double g18 = 1.0 * (-0.5 * nn);         /* mul(-0.5 n, log tau2) */
    g_tau2 += g18 / tau2;                         /* log */
    /* log_det(chol(Q)) with c_bar = 1, then vjp_cholesky(LQ) */
    double* lbq = zalloc(n * w);
    vjp_log_det1(n, bw, LQ, 1.0, lbq);
    double* qbar = zalloc(n * w);
    vjp_chol1(n, bw, LQ, lbq, qbar);              /* accumulate_sym(q): 0 + qbar */
    /* neg(log_det(Lp)): c_bar = -1 */
    double* glp = zalloc(n * w);
    vjp_log_det1(n, bw, Lp, -1.0, glp);
    /* solve_vec(Lp, y): accumulate l_bar into glp */
    double* lbs = zalloc(n * w);
    double* vb = zalloc(n);
    st = vjp_solve_vec1(n, bw, Lp, wv, gw, 0, lbs, vb, row);
    if (st) {
      free(gw); free(lbq); free(qbar); free(glp); free(lbs); free(vb);
      goto done;
    }
    for (ix c = 0; c < n * w; ++c) glp[c] += lbs[c];
    /* cholesky(A) */
    double* abar = zalloc(n * w);
    vjp_chol1(n, bw, Lp, glp, abar);
    for (ix c = 0; c < n * w; ++c) qbar[c] += abar[c]; /* add_diagonal_sym -> q */
    {
      band ab = mk(n, bw, 0, abar);
      double gd = 0.0;                                   /* scale_vec: dot(grad, mask) */
      for (ix i = 0; i < n; ++i) gd += *at(&ab, i, i) * 1.0;
      g_inv += gd;
    }
    g_tau2 += -g_inv * 1.0 / (tau2 * tau2); /* div(1, tau2) */
    *tau2_bar = g_tau2;

    /* chain Q_bar (stored cells, band (bw,0)) through Q = band(L L^T) */
    band G = mk(n, bw, 0, qbar);
    band abar_l = alloc_band(n, bw, 0), bbar_l = alloc_band(n, 0, bw);
    vjp_product1(&Lb, &Lt, &G, &abar_l, &bbar_l);
    band bbt = transpose1(&bbar_l);
    band out = mk(n, bw, 0, lbar_out);
    for (ix j = 0; j < n; ++j) { /* bandgm::add, banded.cpp:122-132 */
      const ix i1 = imin(n - 1, j + bw);
      for (ix i = j; i <= i1; ++i) *at(&out, i, j) = at_or_zero(&abar_l, i, j) + at_or_zero(&bbt, i, j);
    }
    free(abar_l.d); free(bbar_l.d); free(bbt.d);
    free(gw); free(lbq); free(qbar); free(glp); free(lbs); free(vb); free(abar);
  }
done:
  free(Lt.d); free(Q.d); free(A.d); free(Lp); free(LQ); free(wv);
  return st;
}

/* ------------------------------------------------------ batched C ABI */
/* Each batched entry point loops over matrices; `status`/`row` are per
 * matrix (row = -1 when the matrix succeeded). */

#define BATCH_LOOP for (ix b = 0; b < batch; ++b)
#define PAR _Pragma("omp parallel for schedule(dynamic)")

int orc_cholesky(ix batch, ix n, ix bw, const double* q, double* l, int32_t* status, ix* row) {
  const ix w = bw + 1;
  PAR BATCH_LOOP {
    row[b] = -1;
    status[b] = chol1(n, bw, q + b * n * w, l + b * n * w, &row[b]);
  }
  return 0;
}

int orc_solve_vec(ix batch, ix n, ix bw, const double* l, const double* v, int tr, double* x,
                  int32_t* status, ix* row) {
  const ix w = bw + 1;
  PAR BATCH_LOOP {
    row[b] = -1;
    status[b] = solve_vec1(n, bw, l + b * n * w, v + b * n, tr, x + b * n, &row[b]);
  }
  return 0;
}

int orc_log_det(ix batch, ix n, ix bw, const double* l, double* out, int32_t* status, ix* row) {
  const ix w = bw + 1;
  PAR BATCH_LOOP {
    row[b] = -1;
    status[b] = log_det1(n, bw, l + b * n * w, out + b, &row[b]);
  }
  return 0;
}

int orc_sparse_inverse_subset(ix batch, ix n, ix bw, const double* l, double* s, int32_t* status,
                              ix* row) {
  const ix w = bw + 1;
  PAR BATCH_LOOP {
    row[b] = -1;
    status[b] = subset1(n, bw, l + b * n * w, s + b * n * w, &row[b]);
  }
  return 0;
}

/* (ol, ou) must already be clipped to n-1 (kernels.cpp:80-81). */
int orc_product_band_band(ix batch, ix n, ix al, ix au, const double* a, ix bl, ix bu,
                          const double* bm, ix ol, ix ou, double* c) {
  PAR BATCH_LOOP {
    band A = mk(n, al, au, (double*)a + b * n * (al + au + 1));
    band B = mk(n, bl, bu, (double*)bm + b * n * (bl + bu + 1));
    band C = mk(n, ol, ou, c + b * n * (ol + ou + 1));
    product1(&A, &B, &C);
  }
  return 0;
}

int orc_product_band_vec(ix batch, ix n, ix bl, ix bu, const double* bm, const double* v, int tr,
                         double* y) {
  PAR BATCH_LOOP {
    band B = mk(n, bl, bu, (double*)bm + b * n * (bl + bu + 1));
    band_vec1(&B, v + b * n, tr, y + b * n);
  }
  return 0;
}

int orc_outer_band(ix batch, ix n, const double* m, const double* v, ix lo, ix up, double* out) {
  PAR BATCH_LOOP {
    band O = mk(n, lo, up, out + b * n * (lo + up + 1));
    outer1(m + b * n, v + b * n, &O);
  }
  return 0;
}

int orc_solve_mat(ix batch, ix n, ix bw, const double* l, ix rl, ix ru, const double* r, ix ol,
                  ix ou, int tr, double* out, int32_t* status, ix* row) {
  PAR BATCH_LOOP {
    band L = mk(n, bw, 0, (double*)l + b * n * (bw + 1));
    band R = mk(n, rl, ru, (double*)r + b * n * (rl + ru + 1));
    band O = mk(n, ol, ou, out + b * n * (ol + ou + 1));
    row[b] = -1;
    status[b] = solve_mat1(&L, &R, &O, tr, &row[b]);
  }
  return 0;
}

int orc_vjp_cholesky(ix batch, ix n, ix bw, const double* l, const double* lbar, double* qbar) {
  const ix w = bw + 1;
  PAR BATCH_LOOP {
    double* scratch = zalloc(n * w);
    memcpy(scratch, lbar + b * n * w, sizeof(double) * (size_t)(n * w));
    vjp_chol1(n, bw, l + b * n * w, scratch, qbar + b * n * w);
    free(scratch);
  }
  return 0;
}

int orc_vjp_solve_vec(ix batch, ix n, ix bw, const double* l, const double* s, const double* sbar,
                      int tr, double* lbar, double* vbar, int32_t* status, ix* row) {
  const ix w = bw + 1;
  PAR BATCH_LOOP {
    row[b] = -1;
    status[b] = vjp_solve_vec1(n, bw, l + b * n * w, s + b * n, sbar + b * n, tr, lbar + b * n * w,
                               vbar + b * n, &row[b]);
  }
  return 0;
}

int orc_vjp_sparse_inverse_subset(ix batch, ix n, ix bw, const double* l, const double* s,
                                  const double* sbar, double* lbar, int32_t* status, ix* row) {
  const ix w = bw + 1;
  PAR BATCH_LOOP {
    row[b] = -1;
    status[b] = vjp_subset1(n, bw, l + b * n * w, s + b * n * w, sbar + b * n * w, lbar + b * n * w,
                            &row[b]);
  }
  return 0;
}

/* p_bar carries the (already clipped) forward output band (pl, pu). */
int orc_vjp_product_band_band(ix batch, ix n, ix al, ix au, const double* a, ix bl, ix bu,
                              const double* bm, ix pl, ix pu, const double* pbar, double* abar,
                              double* bbar) {
  PAR BATCH_LOOP {
    band A = mk(n, al, au, (double*)a + b * n * (al + au + 1));
    band B = mk(n, bl, bu, (double*)bm + b * n * (bl + bu + 1));
    band P = mk(n, pl, pu, (double*)pbar + b * n * (pl + pu + 1));
    band AB = mk(n, al, au, abar + b * n * (al + au + 1));
    band BB = mk(n, bl, bu, bbar + b * n * (bl + bu + 1));
    vjp_product1(&A, &B, &P, &AB, &BB);
  }
  return 0;
}

/* grad.cpp:153-162 */
int orc_vjp_product_band_vec(ix batch, ix n, ix bl, ix bu, const double* bm, const double* v,
                             const double* pbar, int tr, double* bbar, double* vbar) {
  PAR BATCH_LOOP {
    band B = mk(n, bl, bu, (double*)bm + b * n * (bl + bu + 1));
    band BB = mk(n, bl, bu, bbar + b * n * (bl + bu + 1));
    band_vec1(&B, pbar + b * n, !tr, vbar + b * n);
    if (!tr)
      outer1(pbar + b * n, v + b * n, &BB);
    else
      outer1(v + b * n, pbar + b * n, &BB);
  }
  return 0;
}

/* grad.cpp:164-170 */
int orc_vjp_outer_band(ix batch, ix n, const double* m, const double* v, ix ol, ix ou,
                       const double* obar, double* mbar, double* vbar) {
  PAR BATCH_LOOP {
    band O = mk(n, ol, ou, (double*)obar + b * n * (ol + ou + 1));
    band_vec1(&O, v + b * n, 0, mbar + b * n);
    band_vec1(&O, m + b * n, 1, vbar + b * n);
  }
  return 0;
}

int orc_vjp_log_det(ix batch, ix n, ix bw, const double* l, const double* cbar, double* lbar) {
  const ix w = bw + 1;
  PAR BATCH_LOOP vjp_log_det1(n, bw, l + b * n * w, cbar[b], lbar + b * n * w);
  return 0;
}

/* s / s_bar carry the forward output band (sl, su); r band (rl, ru). */
int orc_vjp_solve_mat(ix batch, ix n, ix bw, const double* l, ix sl, ix su, const double* s,
                      const double* sbar, ix rl, ix ru, int tr, double* lbar, double* rbar,
                      int32_t* status, ix* row) {
  const ix rlc = imin(rl, n - 1), ruc = imin(ru, n - 1);
  PAR BATCH_LOOP {
    band L = mk(n, bw, 0, (double*)l + b * n * (bw + 1));
    band S = mk(n, sl, su, (double*)s + b * n * (sl + su + 1));
    band SB = mk(n, sl, su, (double*)sbar + b * n * (sl + su + 1));
    band LB = mk(n, bw, 0, lbar + b * n * (bw + 1));
    band RB = mk(n, rlc, ruc, rbar + b * n * (rlc + ruc + 1));
    row[b] = -1;
    status[b] = vjp_solve_mat1(&L, &S, &SB, rl, ru, tr, &LB, &RB, &row[b]);
  }
  return 0;
}

int orc_marginal_likelihood_grad(ix batch, ix n, ix bw, const double* L, const double* y,
                                 double tau2, double* loss, double* lbar, double* tau2_bar,
                                 int32_t* status, ix* row) {
  const ix w = bw + 1;
  PAR BATCH_LOOP {
    row[b] = -1;
    status[b] = mlik1(n, bw, L + b * n * w, y + b * n, tau2, loss + b, lbar + b * n * w,
                      tau2_bar + b, &row[b]);
  }
  return 0;
}

int orc_abi_version(void) { return 1; }

/* ------------------------------------------------------------------------
 * Accuracy yardstick (tests only): the config-3 quantities along the banded
 * route in x87 long double (64-bit mantissa) -- the same mathematics as
 * tests/exact.py (and bgm_mlik.cu's header), in C so that the full config-3
 * size (n = 65536) takes seconds:
 *   A = band(L L^T) + I/tau2 = Lp Lp^T, w = Lp^-1 y, u = Lp^-T w,
 *   S = band(A^-1) by the Takahashi recursion (kernels_serial.cpp:80-104),
 *   L_bar = -band_lower[(S + u u^T / tau2^2) L] + diag(1/L_ii),
 *   loss and d tau2 as inference.cpp:140-163 differentiated.
 * Outputs are rounded to double.  One matrix at a time, reference layout.
 * ---------------------------------------------------------------------- */
typedef long double ld_t;

static void mlik_exact1(ix n, ix k, const double* L, const double* y, double tau2, double* loss,
                        double* lbar, double* tbar) {
  const ix w = k + 1;
  const ld_t s = 1.0L / (ld_t)tau2, c4 = s * s;
  ld_t* A = (ld_t*)calloc((size_t)(n * w), sizeof(ld_t));
  ld_t* P = (ld_t*)calloc((size_t)(n * w), sizeof(ld_t));
  ld_t* S = (ld_t*)calloc((size_t)(n * w), sizeof(ld_t));
  ld_t* wv = (ld_t*)calloc((size_t)n, sizeof(ld_t));
  ld_t* u = (ld_t*)calloc((size_t)n, sizeof(ld_t));
#define LL(i, j) ((ld_t)L[(j) * w + ((i) - (j))]) /* lower band entry, i - j in [0, k] */
#define AA(i, j) A[(j) * w + ((i) - (j))]
#define PP(i, j) P[(j) * w + ((i) - (j))]
#define SS(i, j) S[(j) * w + ((i) - (j))]
  for (ix j = 0; j < n; ++j) /* A = band(L L^T) + s I */
    for (ix r = 0; r < w && j + r < n; ++r) {
      const ix i = j + r;
      ld_t acc = 0;
      for (ix m = imax(0, i - k); m <= j; ++m) acc += LL(i, m) * LL(j, m);
      AA(i, j) = acc + (r == 0 ? s : 0);
    }
  for (ix i = 0; i < n; ++i) { /* Cholesky, kernels_serial.cpp:12-32 order */
    const ix j0 = imax(0, i - k);
    for (ix j = j0; j <= i; ++j) {
      ld_t acc = 0;
      for (ix m = j0; m < j; ++m) acc += PP(i, m) * PP(j, m);
      if (i == j) PP(i, i) = sqrtl(AA(i, i) - acc);
      else PP(i, j) = (AA(i, j) - acc) / PP(j, j);
    }
  }
  for (ix i = 0; i < n; ++i) {
    ld_t acc = 0;
    for (ix m = imax(0, i - k); m < i; ++m) acc += PP(i, m) * wv[m];
    wv[i] = ((ld_t)y[i] - acc) / PP(i, i);
  }
  for (ix i = n - 1; i >= 0; --i) {
    ld_t acc = 0;
    for (ix m = i + 1; m < imin(n, i + k + 1); ++m) acc += PP(m, i) * u[m];
    u[i] = (wv[i] - acc) / PP(i, i);
  }
  for (ix j = n - 1; j >= 0; --j) /* Takahashi */
    for (ix i = j; i >= imax(0, j - k); --i) {
      ld_t acc = 0;
      for (ix m = i + 1; m < imin(n, i + k + 1); ++m) {
        const ld_t smj = m >= j ? SS(m, j) : SS(j, m);
        acc += (PP(m, i) / PP(i, i)) * smj;
      }
      SS(j, i) = -acc + (i == j ? 1.0L / (PP(i, i) * PP(i, i)) : 0);
    }
  ld_t yy = 0, ww = 0, uu = 0, tr = 0, ldp = 0, ldl = 0;
  for (ix j = 0; j < n; ++j) {
    for (ix r = 0; r < w; ++r) {
      const ix i = j + r;
      if (i >= n) {
        lbar[j * w + r] = 0.0;
        continue;
      }
      ld_t acc = 0;
      for (ix m = j; m < imin(n, j + k + 1); ++m) {
        const ix d = i > m ? i - m : m - i;
        const ld_t sim = d <= k ? (i >= m ? SS(i, m) : SS(m, i)) : 0;
        acc += sim * LL(m, j) + c4 * u[i] * u[m] * LL(m, j);
      }
      lbar[j * w + r] = (double)(-acc + (r == 0 ? 1.0L / LL(j, j) : 0));
    }
    yy += (ld_t)y[j] * (ld_t)y[j];
    ww += wv[j] * wv[j];
    uu += u[j] * u[j];
    tr += SS(j, j);
    ldp += logl(PP(j, j));
    ldl += logl(fabsl(LL(j, j)));
  }
  const ld_t nn = (ld_t)n, log2pi = 1.837877066409345483560659472811235279722794947275566825634L;
  *loss = (double)(-0.5L * nn * log2pi - ldp + ldl - 0.5L * nn * logl((ld_t)tau2) - 0.5L * yy * s + 0.5L * ww * c4);
  *tbar = (double)(-nn * 0.5L * s + 0.5L * yy * c4 + 0.5L * c4 * tr - ww * c4 * s + 0.5L * uu * c4 * c4);
#undef LL
#undef AA
#undef PP
#undef SS
  free(A);
  free(P);
  free(S);
  free(wv);
  free(u);
}

int orc_mlik_exact_ld(ix batch, ix n, ix k, const double* L, const double* y, double tau2, double* loss,
                      double* lbar, double* tbar) {
  for (ix b = 0; b < batch; ++b)
    mlik_exact1(n, k, L + b * n * (k + 1), y + b * n, tau2, loss + b, lbar + b * n * (k + 1), tbar + b);
  return 0;
}
