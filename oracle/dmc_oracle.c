/*
 * dmc_oracle.c — CPU restatement of the reference dmc hot path (pca_qp,
 * n_b = 1).  TEST INFRASTRUCTURE ONLY (see dmc_oracle.h).  Reference paths
 * below are relative to /root/reference/proj.  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off -fopenmp).
 */
#include "dmc_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* ======================================================================== */
/* mesh.cpp                                                                  */
/* ======================================================================== */

/* src/mesh.cpp:60-86: every face contributes both other corners to each
 * corner's list; lists are sorted and deduplicated. Errors are raised in face
 * order, index check before degeneracy check (mesh.cpp:66-75). */
long orc_build_connectivity(const uint32_t* faces, size_t m, uint32_t n, uint32_t* row_ptr,
                            uint32_t* col) {
  if (m == 0) return -ORC_E_INDEX; /* ValidationError("face list is empty") */
  for (size_t t = 0; t < m; ++t) {
    const uint32_t* f = faces + 3 * t;
    for (int j = 0; j < 3; ++j)
      if (f[j] >= n) return -ORC_E_INDEX; /* IndexOutOfRange */
    if (f[0] == f[1] || f[1] == f[2] || f[0] == f[2]) return -ORC_E_INDEX; /* DegenerateFace */
  }
  uint32_t* cnt = calloc((size_t)n + 1, sizeof(uint32_t));
  for (size_t t = 0; t < 3 * m; ++t) cnt[faces[t] + 1] += 2;
  for (uint32_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  uint32_t* fill = malloc(((size_t)n + 1) * sizeof(uint32_t));
  memcpy(fill, cnt, ((size_t)n + 1) * sizeof(uint32_t));
  for (size_t t = 0; t < m; ++t) {
    const uint32_t* f = faces + 3 * t;
    for (int j = 0; j < 3; ++j) {
      col[fill[f[j]]++] = f[(j + 1) % 3];
      col[fill[f[j]]++] = f[(j + 2) % 3];
    }
  }
  long out = 0;
  row_ptr[0] = 0;
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t b = cnt[i], e = cnt[i + 1];
    qsort(col + b, e - b, sizeof(uint32_t), cmp_u32);
    uint32_t start = (uint32_t)out;
    for (uint32_t p = b; p < e; ++p)
      if (p == b || col[p] != col[p - 1]) col[out++] = col[p];
    (void)start;
    row_ptr[i + 1] = (uint32_t)out;
  }
  free(cnt);
  free(fill);
  return out;
}

/* src/mesh.cpp:88-106 */
static int is_connected(uint32_t n, const uint32_t* rp, const uint32_t* col) {
  if (n == 0) return 0;
  char* seen = calloc(n, 1);
  uint32_t* queue = malloc((size_t)n * sizeof(uint32_t));
  size_t head = 0, tail = 0;
  queue[tail++] = 0;
  seen[0] = 1;
  uint32_t visited = 1;
  while (head < tail) {
    uint32_t v = queue[head++];
    for (uint32_t p = rp[v]; p < rp[v + 1]; ++p) {
      uint32_t w = col[p];
      if (!seen[w]) {
        seen[w] = 1;
        ++visited;
        queue[tail++] = w;
      }
    }
  }
  free(seen);
  free(queue);
  return visited == n;
}

/* src/mesh.cpp:108-136 */
int orc_validate(uint32_t n, uint32_t F, const uint32_t* faces, size_t m, const double* ax,
                 const double* ay, const double* az) {
  if (n == 0 || F == 0) return 1;
  if (m == 0) return 2;
  int issues = 0;
  uint32_t* rp = malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* col = malloc(6 * m * sizeof(uint32_t));
  long nnz = orc_build_connectivity(faces, m, n, rp, col);
  if (nnz < 0) {
    issues |= 16;
  } else {
    for (uint32_t i = 0; i < n; ++i)
      if (rp[i] == rp[i + 1]) {
        issues |= 4;
        break;
      }
    if (!is_connected(n, rp, col)) issues |= 8;
  }
  free(rp);
  free(col);
  const double* axes[3] = {ax, ay, az};
  for (int a = 0; a < 3; ++a)
    for (size_t t = 0; t < (size_t)n * F; ++t)
      if (!isfinite(axes[a][t])) {
        issues |= 32 << a;
        break;
      }
  return issues;
}

/* ======================================================================== */
/* laplacian.cpp                                                             */
/* ======================================================================== */

/* src/laplacian.cpp:21-37: triplets (i,i,d) and (i,j,-1) [Combinatorial] or
 * (i,i,1), (i,j,-1/d) [Normalized], compressed with sorted inner indices. */
void orc_build_laplacian(uint32_t n, const uint32_t* adj_row, const uint32_t* adj_col, int kind,
                         uint32_t* lrow, uint32_t* lcol, double* lval) {
  uint32_t out = 0;
  lrow[0] = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const double d = (double)(adj_row[i + 1] - adj_row[i]);
    const double diag = kind == 0 ? d : 1.0;
    const double off = kind == 0 ? -1.0 : -1.0 / d;
    int placed = 0;
    for (uint32_t p = adj_row[i]; p < adj_row[i + 1]; ++p) {
      if (!placed && adj_col[p] > i) {
        lcol[out] = i;
        lval[out++] = diag;
        placed = 1;
      }
      lcol[out] = adj_col[p];
      lval[out++] = off;
    }
    if (!placed) {
      lcol[out] = i;
      lval[out++] = diag;
    }
    lrow[i + 1] = out;
  }
}

/* src/laplacian.cpp:39-46 — Eigen's ColMajor sparse * dense product adds
 * L(i,j) * x_j into res(i,c) for j ascending, starting from zero. */
void orc_delta(uint32_t n, uint32_t F, const uint32_t* lrow, const uint32_t* lcol,
               const double* lval, const double* X, double* out) {
  for (uint32_t i = 0; i < n; ++i) {
    double* o = out + (size_t)i * F;
    for (uint32_t f = 0; f < F; ++f) o[f] = 0.0;
    for (uint32_t p = lrow[i]; p < lrow[i + 1]; ++p) {
      const double v = lval[p];
      const double* x = X + (size_t)lcol[p] * F;
      for (uint32_t f = 0; f < F; ++f) o[f] = o[f] + v * x[f];
    }
  }
}

/* ======================================================================== */
/* spectral.cpp                                                              */
/* ======================================================================== */

/* src/spectral.cpp:35-39.  Each R(f,g) is summed over vertices in ascending
 * order; R(f,g) and R(g,f) are computed identically, so the symmetrisation
 * 0.5*(R+R^T) is exact and reduces to mirroring. */
void orc_autocorrelation(uint32_t n, uint32_t F, const double* X, double* R) {
  memset(R, 0, (size_t)F * F * sizeof(double));
  for (uint32_t i = 0; i < n; ++i) {
    const double* x = X + (size_t)i * F;
    for (uint32_t g = 0; g < F; ++g) {
      const double xg = x[g];
      double* rc = R + (size_t)g * F; /* column g, rows f <= g */
      for (uint32_t f = 0; f <= g; ++f) rc[f] = rc[f] + x[f] * xg;
    }
  }
  for (uint32_t g = 0; g < F; ++g)
    for (uint32_t f = 0; f < g; ++f) R[(size_t)f * F + g] = R[(size_t)g * F + f];
}

/* src/spectral.cpp:41-47: Eigen's maxCoeff(&idx) keeps the first maximal
 * index; a negative entry there flips the column. */
void orc_canonicalize_signs(uint32_t m, uint32_t p, double* U) {
  for (uint32_t j = 0; j < p; ++j) {
    double* c = U + (size_t)j * m;
    uint32_t imax = 0;
    double best = fabs(c[0]);
    for (uint32_t i = 1; i < m; ++i)
      if (fabs(c[i]) > best) {
        best = fabs(c[i]);
        imax = i;
      }
    if (c[imax] < 0.0)
      for (uint32_t i = 0; i < m; ++i) c[i] = -c[i];
  }
}

/* Round-robin ("chess tournament") pairing of step s of a sweep over m2
 * (even) indices; identical on the GPU (csrc/basis.cu). */
static void rr_pair(uint32_t m2, uint32_t s, uint32_t i, uint32_t* p, uint32_t* q) {
  uint32_t a, b;
  const uint32_t r = m2 - 1;
  if (i == 0) {
    a = 0;
    b = (s + r - 1) % r + 1;
  } else {
    a = (i + s - 1) % r + 1;
    b = (r - i + s - 1) % r + 1;
  }
  *p = a < b ? a : b;
  *q = a < b ? b : a;
}

/* Jacobi rotation for the 2x2 block [[app, apq], [apq, aqq]] (Rutishauser).
 * Returns 0 when the pair is skipped. */
static int jacobi_rot(double app, double aqq, double apq, double thresh, double* c, double* s,
                      double* t) {
  if (!(fabs(apq) > thresh)) return 0;
  const double theta = (aqq - app) / (2.0 * apq);
  double tt;
  if (fabs(theta) > 1e150)
    tt = 0.5 / theta;
  else
    tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
  const double cc = 1.0 / sqrt(tt * tt + 1.0);
  *c = cc;
  *s = tt * cc;
  *t = tt;
  return 1;
}

int orc_jacobi_eig(uint32_t m, double* A_in, double* V_out, double* w) {
  const uint32_t m2 = m + (m & 1u);
  double* A = calloc((size_t)m2 * m2, sizeof(double));
  double* V = calloc((size_t)m2 * m2, sizeof(double));
  for (uint32_t j = 0; j < m; ++j)
    for (uint32_t i = 0; i < m; ++i) A[(size_t)j * m2 + i] = A_in[(size_t)j * m + i];
  for (uint32_t i = 0; i < m2; ++i) V[(size_t)i * m2 + i] = 1.0;
  double fro = 0.0;
  for (size_t t = 0; t < (size_t)m2 * m2; ++t) fro += A[t] * A[t];
  fro = sqrt(fro);
  const double abs_thresh = fro * 1e-22 + DBL_MIN;
  const uint32_t h = m2 / 2;
  double *cs = malloc(h * sizeof(double)), *sn = malloc(h * sizeof(double)),
         *tn = malloc(h * sizeof(double));
  uint32_t *P = malloc(h * sizeof(uint32_t)), *Q = malloc(h * sizeof(uint32_t));
  char* act = malloc(h);
  int sweep, converged = 0;
  for (sweep = 0; sweep < 60 && m2 > 1; ++sweep) {
    long rotations = 0;
    for (uint32_t s = 0; s + 1 < m2; ++s) {
      for (uint32_t i = 0; i < h; ++i) {
        rr_pair(m2, s, i, &P[i], &Q[i]);
        const double app = A[(size_t)P[i] * m2 + P[i]], aqq = A[(size_t)Q[i] * m2 + Q[i]];
        const double apq = A[(size_t)Q[i] * m2 + P[i]];
        const double rel = 1e-17 * sqrt(fabs(app) * fabs(aqq));
        act[i] = (char)jacobi_rot(app, aqq, apq, rel > abs_thresh ? rel : abs_thresh, &cs[i],
                                  &sn[i], &tn[i]);
        if (!act[i]) {
          cs[i] = 1.0;
          sn[i] = 0.0;
          tn[i] = 0.0;
        }
        rotations += act[i];
      }
      /* A <- J^T A J, block by block over pair indices a <= b. */
      for (uint32_t a = 0; a < h; ++a)
        for (uint32_t b = a; b < h; ++b) {
          const uint32_t p1 = P[a], q1 = Q[a], p2 = P[b], q2 = Q[b];
          if (a == b) {
            const double apq = A[(size_t)q1 * m2 + p1];
            if (act[a]) {
              A[(size_t)p1 * m2 + p1] = A[(size_t)p1 * m2 + p1] - tn[a] * apq;
              A[(size_t)q1 * m2 + q1] = A[(size_t)q1 * m2 + q1] + tn[a] * apq;
              A[(size_t)q1 * m2 + p1] = 0.0;
              A[(size_t)p1 * m2 + q1] = 0.0;
            }
            continue;
          }
          if (!act[a] && !act[b]) continue;
          const double ca = cs[a], sa = sn[a], cb = cs[b], sb = sn[b];
          const double b00 = A[(size_t)p2 * m2 + p1], b01 = A[(size_t)q2 * m2 + p1];
          const double b10 = A[(size_t)p2 * m2 + q1], b11 = A[(size_t)q2 * m2 + q1];
          const double r00 = ca * b00 - sa * b10, r01 = ca * b01 - sa * b11;
          const double r10 = sa * b00 + ca * b10, r11 = sa * b01 + ca * b11;
          const double n00 = cb * r00 - sb * r01, n01 = sb * r00 + cb * r01;
          const double n10 = cb * r10 - sb * r11, n11 = sb * r10 + cb * r11;
          A[(size_t)p2 * m2 + p1] = n00;
          A[(size_t)p1 * m2 + p2] = n00;
          A[(size_t)q2 * m2 + p1] = n01;
          A[(size_t)p1 * m2 + q2] = n01;
          A[(size_t)p2 * m2 + q1] = n10;
          A[(size_t)q1 * m2 + p2] = n10;
          A[(size_t)q2 * m2 + q1] = n11;
          A[(size_t)q1 * m2 + q2] = n11;
        }
      /* V <- V J */
      for (uint32_t a = 0; a < h; ++a) {
        if (!act[a]) continue;
        double* vp = V + (size_t)P[a] * m2;
        double* vq = V + (size_t)Q[a] * m2;
        const double c = cs[a], sv = sn[a];
        for (uint32_t r = 0; r < m2; ++r) {
          const double x = vp[r], y = vq[r];
          vp[r] = c * x - sv * y;
          vq[r] = sv * x + c * y;
        }
      }
    }
    if (rotations == 0) {
      converged = 1;
      break;
    }
  }
  if (m2 <= 1) converged = 1;
  for (uint32_t j = 0; j < m; ++j) {
    w[j] = A[(size_t)j * m2 + j];
    for (uint32_t i = 0; i < m; ++i) V_out[(size_t)j * m + i] = V[(size_t)j * m2 + i];
  }
  (void)A_in;
  free(A);
  free(V);
  free(cs);
  free(sn);
  free(tn);
  free(P);
  free(Q);
  free(act);
  return converged ? sweep : -ORC_E_NUMERICAL;
}

/* Stable descending order of w (ties keep the lower index first). */
static void order_desc(uint32_t m, const double* w, uint32_t* idx) {
  for (uint32_t i = 0; i < m; ++i) idx[i] = i;
  for (uint32_t i = 1; i < m; ++i) { /* insertion sort, stable */
    uint32_t v = idx[i];
    int j = (int)i - 1;
    while (j >= 0 && w[idx[j]] < w[v]) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = v;
  }
}

/* src/spectral.cpp:49-67 */
int orc_full_eigenbasis(uint32_t m, const double* R, double* U, double* evals) {
  double* A = malloc((size_t)m * m * sizeof(double));
  double* V = malloc((size_t)m * m * sizeof(double));
  double* w = malloc((size_t)m * sizeof(double));
  uint32_t* idx = malloc((size_t)m * sizeof(uint32_t));
  memcpy(A, R, (size_t)m * m * sizeof(double));
  int rc = orc_jacobi_eig(m, A, V, w);
  if (rc >= 0) {
    order_desc(m, w, idx);
    for (uint32_t j = 0; j < m; ++j) {
      memcpy(U + (size_t)j * m, V + (size_t)idx[j] * m, (size_t)m * sizeof(double));
      if (evals) evals[j] = w[idx[j]];
    }
    orc_canonicalize_signs(m, m, U);
  }
  free(A);
  free(V);
  free(w);
  free(idx);
  return rc >= 0 ? 0 : ORC_E_NUMERICAL;
}

/* Householder QR in place (Eigen::HouseholderQR / makeHouseholder):
 * beta = -sign(c0) * ||x||, tau = (beta - c0) / beta, v = [1; tail/(c0-beta)];
 * a vanishing tail (||tail||^2 <= DBL_MIN) gives tau = 0, beta = c0.
 * Z (m x p, col-major) is overwritten with the essential parts below the
 * diagonal; betas (R diagonal) and taus are returned. */
static void householder_factor(uint32_t m, uint32_t p, double* Z, double* tau, double* beta) {
  for (uint32_t j = 0; j < p && j < m; ++j) {
    double* x = Z + (size_t)j * m;
    const double c0 = x[j];
    double tail = 0.0;
    for (uint32_t i = j + 1; i < m; ++i) tail += x[i] * x[i];
    if (tail <= DBL_MIN) {
      tau[j] = 0.0;
      beta[j] = c0;
      for (uint32_t i = j + 1; i < m; ++i) x[i] = 0.0;
      continue;
    }
    double b = sqrt(c0 * c0 + tail);
    if (c0 >= 0.0) b = -b;
    const double denom = c0 - b;
    for (uint32_t i = j + 1; i < m; ++i) x[i] = x[i] / denom;
    tau[j] = (b - c0) / b;
    beta[j] = b;
    x[j] = b;
    /* apply H_j = I - tau v v^T to trailing columns */
    for (uint32_t c = j + 1; c < p; ++c) {
      double* y = Z + (size_t)c * m;
      double d = y[j];
      for (uint32_t i = j + 1; i < m; ++i) d += x[i] * y[i];
      d = tau[j] * d;
      y[j] = y[j] - d;
      for (uint32_t i = j + 1; i < m; ++i) y[i] = y[i] - d * x[i];
    }
  }
}

/* Applies H_0 ... H_{p-1} (factored in F) to the m x q matrix B in place. */
static void householder_apply(uint32_t m, uint32_t p, const double* F_, const double* tau,
                              double* B, uint32_t q) {
  for (int j = (int)p - 1; j >= 0; --j) {
    if (tau[j] == 0.0) continue;
    const double* v = F_ + (size_t)j * m;
    for (uint32_t c = 0; c < q; ++c) {
      double* y = B + (size_t)c * m;
      double d = y[j];
      for (uint32_t i = j + 1; i < m; ++i) d += v[i] * y[i];
      d = tau[j] * d;
      y[j] = y[j] - d;
      for (uint32_t i = j + 1; i < m; ++i) y[i] = y[i] - d * v[i];
    }
  }
}

void orc_householder_q(uint32_t m, uint32_t p, const double* Z, double* Q) {
  double* W = malloc((size_t)m * p * sizeof(double));
  double* tau = malloc((size_t)p * sizeof(double));
  double* beta = malloc((size_t)p * sizeof(double));
  memcpy(W, Z, (size_t)m * p * sizeof(double));
  householder_factor(m, p, W, tau, beta);
  memset(Q, 0, (size_t)m * p * sizeof(double));
  for (uint32_t j = 0; j < p; ++j) Q[(size_t)j * m + j] = 1.0;
  householder_apply(m, p, W, tau, Q, p);
  free(W);
  free(tau);
  free(beta);
}

/* C (m x q) = A (m x k) * B (k x q), all column-major, ascending-k sums. */
static void gemm_nn(uint32_t m, uint32_t k, uint32_t q, const double* A, const double* B,
                    double* C) {
  for (uint32_t c = 0; c < q; ++c) {
    double* o = C + (size_t)c * m;
    for (uint32_t i = 0; i < m; ++i) o[i] = 0.0;
    for (uint32_t t = 0; t < k; ++t) {
      const double b = B[(size_t)c * k + t];
      const double* a = A + (size_t)t * m;
      for (uint32_t i = 0; i < m; ++i) o[i] = o[i] + a[i] * b;
    }
  }
}

/* src/spectral.cpp:69-104 */
int orc_orthogonal_iterations(uint32_t m, const double* R, const double* U_init, int t_max,
                              double stop_tol, double* U_out) {
  if (t_max < 1) return ORC_E_CONFIG;
  double* U = malloc((size_t)m * m * sizeof(double));
  double* Z = malloc((size_t)m * m * sizeof(double));
  double* N = malloc((size_t)m * m * sizeof(double));
  double* tau = malloc((size_t)m * sizeof(double));
  double* beta = malloc((size_t)m * sizeof(double));
  memcpy(U, U_init, (size_t)m * m * sizeof(double));
  int rc = 0;
  for (int t = 2; t <= t_max; ++t) {
    gemm_nn(m, m, m, R, U, Z);
    householder_factor(m, m, Z, tau, beta);
    double mx = 0.0;
    for (uint32_t j = 0; j < m; ++j)
      if (fabs(beta[j]) > mx) mx = fabs(beta[j]);
    const double tol = (double)m * DBL_EPSILON * mx;
    for (uint32_t j = 0; j < m; ++j)
      if (fabs(beta[j]) <= tol) rc = ORC_E_NUMERICAL; /* RankDeficiency */
    if (rc) break;
    memset(N, 0, (size_t)m * m * sizeof(double));
    for (uint32_t j = 0; j < m; ++j) N[(size_t)j * m + j] = 1.0;
    householder_apply(m, m, Z, tau, N, m);
    if (stop_tol >= 0.0) {
      double moved = 0.0;
      for (uint32_t j = 0; j < m; ++j) {
        double d = 0.0;
        for (uint32_t i = 0; i < m; ++i) d += U[(size_t)j * m + i] * N[(size_t)j * m + i];
        double c = fabs(d);
        if (c > 1.0) c = 1.0;
        const double ang = acos(c);
        if (ang > moved) moved = ang;
      }
      memcpy(U, N, (size_t)m * m * sizeof(double));
      if (moved < stop_tol) break;
    } else {
      memcpy(U, N, (size_t)m * m * sizeof(double));
    }
  }
  if (!rc) {
    orc_canonicalize_signs(m, m, U);
    memcpy(U_out, U, (size_t)m * m * sizeof(double));
  }
  free(U);
  free(Z);
  free(N);
  free(tau);
  free(beta);
  return rc;
}

static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void orc_start_matrix(uint64_t seed, size_t count, double* out) {
  uint64_t s = seed;
  for (size_t i = 0; i < count; ++i)
    out[i] = (double)(splitmix64(&s) >> 11) * 0x1.0p-52 - 1.0;
}

int orc_basis(uint32_t F, uint32_t k, const double* R, int rounds, uint64_t seed, double* U,
              double* evals) {
  if (rounds <= 0 || k >= F || k == 0) {
    /* rounds == 0: the reference's n_b = 1 path, codec.cpp:158-159. */
    return orc_full_eigenbasis(F, R, U, evals);
  }
  double* Q = malloc((size_t)F * k * sizeof(double));
  double* Z = malloc((size_t)F * k * sizeof(double));
  double* H = malloc((size_t)k * k * sizeof(double));
  double* W = malloc((size_t)k * k * sizeof(double));
  double* w = malloc((size_t)k * sizeof(double));
  uint32_t* idx = malloc((size_t)k * sizeof(uint32_t));
  double* tau = malloc((size_t)k * sizeof(double));
  double* beta = malloc((size_t)k * sizeof(double));
  orc_start_matrix(seed, (size_t)F * k, Z);
  orc_householder_q(F, k, Z, Q);
  for (int t = 0; t < rounds; ++t) {
    gemm_nn(F, F, k, R, Q, Z);
    orc_householder_q(F, k, Z, Q);
  }
  /* Rayleigh-Ritz: H = Q^T (R Q), symmetrised. */
  gemm_nn(F, F, k, R, Q, Z);
  for (uint32_t j = 0; j < k; ++j)
    for (uint32_t i = 0; i < k; ++i) {
      double d = 0.0;
      for (uint32_t g = 0; g < F; ++g) d = d + Q[(size_t)i * F + g] * Z[(size_t)j * F + g];
      H[(size_t)j * k + i] = d;
    }
  for (uint32_t j = 0; j < k; ++j)
    for (uint32_t i = 0; i < j; ++i) {
      const double s = 0.5 * (H[(size_t)j * k + i] + H[(size_t)i * k + j]);
      H[(size_t)j * k + i] = s;
      H[(size_t)i * k + j] = s;
    }
  int rc = orc_jacobi_eig(k, H, W, w);
  if (rc < 0) goto done;
  rc = 0;
  order_desc(k, w, idx);
  /* U[:, j] = Q W[:, idx[j]] */
  for (uint32_t j = 0; j < k; ++j) {
    const double* wc = W + (size_t)idx[j] * k;
    double* o = U + (size_t)j * F;
    for (uint32_t g = 0; g < F; ++g) o[g] = 0.0;
    for (uint32_t t = 0; t < k; ++t) {
      const double b = wc[t];
      const double* a = Q + (size_t)t * F;
      for (uint32_t g = 0; g < F; ++g) o[g] = o[g] + a[g] * b;
    }
    if (evals) evals[j] = w[idx[j]];
  }
  orc_canonicalize_signs(F, k, U);
  /* Completion: columns k..F-1 of the full Householder Q of U[:, :k]. */
  {
    double* Fk = malloc((size_t)F * k * sizeof(double));
    memcpy(Fk, U, (size_t)F * k * sizeof(double));
    householder_factor(F, k, Fk, tau, beta);
    double* C = U + (size_t)k * F;
    memset(C, 0, (size_t)F * (F - k) * sizeof(double));
    for (uint32_t j = k; j < F; ++j) C[(size_t)(j - k) * F + j] = 1.0;
    householder_apply(F, k, Fk, tau, C, F - k);
    orc_canonicalize_signs(F, F - k, C);
    if (evals)
      for (uint32_t j = k; j < F; ++j) evals[j] = 0.0;
    free(Fk);
  }
done:
  free(Q);
  free(Z);
  free(H);
  free(W);
  free(w);
  free(idx);
  free(tau);
  free(beta);
  return rc;
}

/* src/spectral.cpp:133-140 */
double orc_subspace_angle(uint32_t m, uint32_t p, const double* U, const double* V) {
  double* M = malloc((size_t)p * p * sizeof(double));
  double* G = malloc((size_t)p * p * sizeof(double));
  double* E = malloc((size_t)p * p * sizeof(double));
  double* w = malloc((size_t)p * sizeof(double));
  for (uint32_t j = 0; j < p; ++j)
    for (uint32_t i = 0; i < p; ++i) {
      double d = 0.0;
      for (uint32_t g = 0; g < m; ++g) d += U[(size_t)i * m + g] * V[(size_t)j * m + g];
      M[(size_t)j * p + i] = d;
    }
  for (uint32_t j = 0; j < p; ++j)
    for (uint32_t i = 0; i < p; ++i) {
      double d = 0.0;
      for (uint32_t g = 0; g < p; ++g) d += M[(size_t)i * p + g] * M[(size_t)j * p + g];
      G[(size_t)j * p + i] = d;
    }
  orc_jacobi_eig(p, G, E, w);
  double mn = INFINITY;
  for (uint32_t j = 0; j < p; ++j)
    if (w[j] < mn) mn = w[j];
  double smin = sqrt(mn > 0.0 ? mn : 0.0);
  if (smin > 1.0) smin = 1.0;
  free(M);
  free(G);
  free(E);
  free(w);
  return acos(smin);
}

/* ======================================================================== */
/* quantize.cpp / codec.cpp                                                  */
/* ======================================================================== */

/* src/codec.cpp:31-41 */
void orc_widened_range(double lo, double hi, float* flo, float* fhi) {
  float a = (float)lo;
  if ((double)a > lo) a = nextafterf(a, -INFINITY);
  float b = (float)hi;
  if ((double)b < hi) b = nextafterf(b, INFINITY);
  *flo = a;
  *fhi = b;
}

/* src/quantize.cpp:22-29 */
uint32_t orc_quantize(float mn, float mx, int bits, double x) {
  const uint32_t levels = 1u << bits;
  if (mn == mx) return 0;
  const double min_ = (double)mn;
  const double width = ((double)mx - min_) / levels;
  const double t = floor((x - min_) / width);
  if (t <= 0.0) return 0;
  if (t >= (double)(levels - 1)) return levels - 1;
  return (uint32_t)t;
}

/* src/quantize.cpp:31-38 (level range checked by callers) */
double orc_dequantize(float mn, float mx, int bits, uint32_t level) {
  const uint32_t levels = 1u << bits;
  const double min_ = (double)mn;
  if (mn == mx) return min_;
  const double width = ((double)mx - min_) / levels;
  return min_ + ((double)level + 0.5) * width;
}

/* src/codec.cpp:199-202 */
uint32_t orc_anchor_count(uint32_t n, double fraction) {
  long long r = llround(fraction * n);
  if (r < 1) r = 1;
  if (r > (long long)n) r = n;
  return (uint32_t)r;
}

/* MT19937-64 (Matsumoto & Nishimura), the engine std::mt19937_64 specifies. */
typedef struct {
  uint64_t mt[312];
  int mti;
} mt64;
static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = 312;
}
static uint64_t mt64_next(mt64* g) {
  static const uint64_t mag01[2] = {0ull, 0xB5026F5AA96619E9ull};
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (g->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ull)];
    }
    for (; i < 311; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ull)];
    }
    x = (g->mt[311] & UM) | (g->mt[0] & LM);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ull)];
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

/* src/codec.cpp:204-242 */
int orc_select_anchors(uint32_t n, uint32_t n_c, int strategy, uint64_t seed, uint32_t* out) {
  if (n_c < 1 || n_c > n) return ORC_E_CONFIG; /* InvalidCount */
  if (strategy == 0) {
    uint32_t cnt = 0;
    for (uint64_t j = 0; j < n_c; ++j) out[cnt++] = (uint32_t)(j * n / n_c);
    qsort(out, cnt, sizeof(uint32_t), cmp_u32);
    uint32_t u = 0;
    for (uint32_t i = 0; i < cnt; ++i)
      if (i == 0 || out[i] != out[i - 1]) out[u++] = out[i];
    char* used = calloc(n, 1);
    for (uint32_t i = 0; i < u; ++i) used[out[i]] = 1;
    for (uint32_t i = 0; u < n_c && i < n; ++i)
      if (!used[i]) {
        out[u++] = i;
        used[i] = 1;
      }
    free(used);
    qsort(out, u, sizeof(uint32_t), cmp_u32);
  } else {
    uint32_t* pool = malloc((size_t)n * sizeof(uint32_t));
    for (uint32_t i = 0; i < n; ++i) pool[i] = i;
    mt64 g;
    mt64_seed(&g, seed);
    for (uint32_t i = n - 1; i > 0; --i) {
      const uint64_t j = mt64_next(&g) % ((uint64_t)i + 1);
      uint32_t t = pool[i];
      pool[i] = pool[j];
      pool[j] = t;
    }
    memcpy(out, pool, (size_t)n_c * sizeof(uint32_t));
    qsort(out, n_c, sizeof(uint32_t), cmp_u32);
    free(pool);
  }
  return 0;
}

/* src/codec.cpp:244-265 */
void orc_quantize_rows(uint32_t k_l, uint32_t n, const double* C, const int* row_bits, float* rmin,
                       float* rmax, uint32_t* q) {
  for (uint32_t r = 0; r < k_l; ++r) {
    const double* row = C + (size_t)r * n;
    double lo = row[0], hi = row[0];
    for (uint32_t i = 1; i < n; ++i) {
      if (row[i] < lo) lo = row[i];
      if (row[i] > hi) hi = row[i];
    }
    float flo, fhi;
    orc_widened_range(lo, hi, &flo, &fhi);
    rmin[r] = flo;
    rmax[r] = fhi;
    uint32_t* qr = q + (size_t)r * n;
    for (uint32_t i = 0; i < n; ++i) qr[i] = orc_quantize(flo, fhi, row_bits[r], row[i]);
  }
}

/* src/codec.cpp:267-288 */
int orc_dequantize_rows(uint32_t k_l, uint32_t m, uint32_t n, const float* rmin, const float* rmax,
                        const uint8_t* rbits, const uint32_t* q, double* out) {
  if (k_l > m) return ORC_E_CONFIG;
  memset(out, 0, (size_t)m * n * sizeof(double));
  for (uint32_t r = 0; r < k_l; ++r) {
    double* o = out + (size_t)r * n;
    if (rmin[r] == rmax[r]) {
      for (uint32_t i = 0; i < n; ++i) o[i] = (double)rmin[r];
      continue;
    }
    const uint32_t levels = 1u << rbits[r];
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t lv = q[(size_t)r * n + i];
      if (lv >= levels) return ORC_E_CORRUPT;
      o[i] = orc_dequantize(rmin[r], rmax[r], rbits[r], lv);
    }
  }
  return 0;
}

/* ======================================================================== */
/* solver.cpp                                                                */
/* ======================================================================== */

typedef struct {
  uint32_t n;
  uint32_t *rp, *ci;
  double* v;
} csr;

static void csr_free(csr* a) {
  free(a->rp);
  free(a->ci);
  free(a->v);
}

/* anchored_normal_matrix (src/solver.cpp:25-39): M = L^T L + S^T S. */
static csr normal_matrix(uint32_t n, const uint32_t* lrow, const uint32_t* lcol, const double* lval,
                         uint32_t n_c, const uint32_t* idx) {
  /* L^T: transpose of CSR. */
  uint32_t nnz = lrow[n];
  uint32_t* trp = calloc((size_t)n + 1, sizeof(uint32_t));
  uint32_t* tci = malloc((size_t)nnz * sizeof(uint32_t));
  double* tv = malloc((size_t)nnz * sizeof(double));
  for (uint32_t p = 0; p < nnz; ++p) trp[lcol[p] + 1]++;
  for (uint32_t i = 0; i < n; ++i) trp[i + 1] += trp[i];
  uint32_t* fill = malloc(((size_t)n + 1) * sizeof(uint32_t));
  memcpy(fill, trp, ((size_t)n + 1) * sizeof(uint32_t));
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t p = lrow[i]; p < lrow[i + 1]; ++p) {
      uint32_t d = fill[lcol[p]]++;
      tci[d] = i;
      tv[d] = lval[p];
    }
  free(fill);
  char* anc = calloc(n, 1);
  for (uint32_t a = 0; a < n_c; ++a) anc[idx[a]] = 1;
  /* row i of M = sum_k (L^T)(i,k) * L(k,:) */
  size_t cap = (size_t)nnz * 4 + n;
  csr M;
  M.n = n;
  M.rp = malloc(((size_t)n + 1) * sizeof(uint32_t));
  M.ci = malloc(cap * sizeof(uint32_t));
  M.v = malloc(cap * sizeof(double));
  double* acc = calloc(n, sizeof(double));
  int32_t* mark = malloc((size_t)n * sizeof(int32_t));
  for (uint32_t i = 0; i < n; ++i) mark[i] = -1;
  uint32_t* list = malloc((size_t)n * sizeof(uint32_t));
  size_t out = 0;
  M.rp[0] = 0;
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t cnt = 0;
    for (uint32_t p = trp[i]; p < trp[i + 1]; ++p) {
      const uint32_t k = tci[p];
      const double a = tv[p];
      for (uint32_t q = lrow[k]; q < lrow[k + 1]; ++q) {
        const uint32_t j = lcol[q];
        if (mark[j] != (int32_t)i) {
          mark[j] = (int32_t)i;
          acc[j] = 0.0;
          list[cnt++] = j;
        }
        acc[j] += a * lval[q];
      }
    }
    if (anc[i]) {
      if (mark[i] != (int32_t)i) {
        mark[i] = (int32_t)i;
        acc[i] = 0.0;
        list[cnt++] = i;
      }
      acc[i] += 1.0;
    }
    qsort(list, cnt, sizeof(uint32_t), cmp_u32);
    if (out + cnt > cap) {
      cap = (out + cnt) * 2;
      M.ci = realloc(M.ci, cap * sizeof(uint32_t));
      M.v = realloc(M.v, cap * sizeof(double));
    }
    for (uint32_t t = 0; t < cnt; ++t) {
      M.ci[out] = list[t];
      M.v[out++] = acc[list[t]];
    }
    M.rp[i + 1] = (uint32_t)out;
  }
  free(trp);
  free(tci);
  free(tv);
  free(anc);
  free(acc);
  free(mark);
  free(list);
  return M;
}

/* Fill-reducing ordering: recursive nested dissection by BFS level sets on
 * the graph of M (a level of M's graph is a vertex separator of M). */
typedef struct {
  const csr* M;
  int32_t* part; /* current sub-problem id per vertex */
  int32_t* level;
  uint32_t* queue;
  uint32_t* perm;
  uint32_t nperm;
  int32_t next_id;
} nd_state;

static uint32_t bfs_levels(nd_state* st, const uint32_t* verts, uint32_t cnt, int32_t id,
                           uint32_t root, uint32_t* maxlev) {
  for (uint32_t t = 0; t < cnt; ++t) st->level[verts[t]] = -1;
  uint32_t head = 0, tail = 0;
  st->queue[tail++] = root;
  st->level[root] = 0;
  uint32_t last = root;
  while (head < tail) {
    uint32_t v = st->queue[head++];
    last = v;
    for (uint32_t p = st->M->rp[v]; p < st->M->rp[v + 1]; ++p) {
      uint32_t w = st->M->ci[p];
      if (st->part[w] == id && st->level[w] < 0) {
        st->level[w] = st->level[v] + 1;
        st->queue[tail++] = w;
      }
    }
  }
  *maxlev = (uint32_t)st->level[last];
  return tail; /* vertices reached */
}

static void nd_recurse(nd_state* st, uint32_t* verts, uint32_t cnt, int32_t id) {
  if (cnt == 0) return;
  if (cnt <= 64) {
    for (uint32_t t = 0; t < cnt; ++t) st->perm[st->nperm++] = verts[t];
    return;
  }
  uint32_t maxlev;
  uint32_t reached = bfs_levels(st, verts, cnt, id, verts[0], &maxlev);
  if (reached < cnt) {
    /* disconnected: split off the reached component */
    uint32_t* a = malloc((size_t)reached * sizeof(uint32_t));
    uint32_t* b = malloc((size_t)(cnt - reached) * sizeof(uint32_t));
    uint32_t na = 0, nb = 0;
    for (uint32_t t = 0; t < cnt; ++t) {
      if (st->level[verts[t]] >= 0)
        a[na++] = verts[t];
      else
        b[nb++] = verts[t];
    }
    int32_t ia = st->next_id++, ib = st->next_id++;
    for (uint32_t t = 0; t < na; ++t) st->part[a[t]] = ia;
    for (uint32_t t = 0; t < nb; ++t) st->part[b[t]] = ib;
    nd_recurse(st, a, na, ia);
    nd_recurse(st, b, nb, ib);
    free(a);
    free(b);
    return;
  }
  /* pseudo-peripheral root: restart from the last vertex reached */
  uint32_t root = st->queue[cnt - 1];
  for (int it = 0; it < 2; ++it) {
    uint32_t ml;
    bfs_levels(st, verts, cnt, id, root, &ml);
    if (ml <= maxlev && it > 0) break;
    maxlev = ml;
    root = st->queue[cnt - 1];
  }
  bfs_levels(st, verts, cnt, id, root, &maxlev);
  if (maxlev < 2) {
    for (uint32_t t = 0; t < cnt; ++t) st->perm[st->nperm++] = verts[t];
    return;
  }
  /* pick the separator level closest to half of the vertices */
  uint32_t* hist = calloc((size_t)maxlev + 1, sizeof(uint32_t));
  for (uint32_t t = 0; t < cnt; ++t) hist[st->level[verts[t]]]++;
  uint32_t acc = 0, sep = 1;
  for (uint32_t l = 0; l <= maxlev; ++l) {
    if (acc + hist[l] > cnt / 2) {
      sep = l;
      break;
    }
    acc += hist[l];
  }
  if (sep == 0) sep = 1;
  if (sep >= maxlev) sep = maxlev - 1;
  free(hist);
  uint32_t* a = malloc((size_t)cnt * sizeof(uint32_t));
  uint32_t* b = malloc((size_t)cnt * sizeof(uint32_t));
  uint32_t* s = malloc((size_t)cnt * sizeof(uint32_t));
  uint32_t na = 0, nb = 0, ns = 0;
  for (uint32_t t = 0; t < cnt; ++t) {
    const uint32_t v = verts[t];
    const int32_t l = st->level[v];
    if ((uint32_t)l < sep)
      a[na++] = v;
    else if ((uint32_t)l > sep)
      b[nb++] = v;
    else
      s[ns++] = v;
  }
  int32_t ia = st->next_id++, ib = st->next_id++, is = st->next_id++;
  for (uint32_t t = 0; t < na; ++t) st->part[a[t]] = ia;
  for (uint32_t t = 0; t < nb; ++t) st->part[b[t]] = ib;
  for (uint32_t t = 0; t < ns; ++t) st->part[s[t]] = is;
  nd_recurse(st, a, na, ia);
  nd_recurse(st, b, nb, ib);
  for (uint32_t t = 0; t < ns; ++t) st->perm[st->nperm++] = s[t];
  free(a);
  free(b);
  free(s);
}

/* Sparse LDL^T (up-looking; Davis, ACM TOMS Algorithm 849) of P M P^T. */
typedef struct {
  uint32_t n;
  uint32_t *perm, *pinv;
  size_t* Lp;
  uint32_t* Li;
  double *Lx, *D;
} ldl_factor;

static int ldl_factorize(const csr* M, ldl_factor* f) {
  const uint32_t n = M->n;
  int32_t* parent = malloc((size_t)n * sizeof(int32_t));
  int32_t* flag = malloc((size_t)n * sizeof(int32_t));
  size_t* lnz = calloc(n, sizeof(size_t));
  /* symbolic: elimination tree and column counts */
  for (uint32_t k = 0; k < n; ++k) {
    parent[k] = -1;
    flag[k] = (int32_t)k;
    const uint32_t ko = f->perm[k];
    for (uint32_t p = M->rp[ko]; p < M->rp[ko + 1]; ++p) {
      uint32_t i = f->pinv[M->ci[p]];
      if (i >= k) continue;
      for (; flag[i] != (int32_t)k; i = (uint32_t)parent[i]) {
        if (parent[i] == -1) parent[i] = (int32_t)k;
        lnz[i]++;
        flag[i] = (int32_t)k;
      }
    }
  }
  f->Lp = malloc(((size_t)n + 1) * sizeof(size_t));
  f->Lp[0] = 0;
  for (uint32_t k = 0; k < n; ++k) f->Lp[k + 1] = f->Lp[k] + lnz[k];
  f->Li = malloc((f->Lp[n] + 1) * sizeof(uint32_t));
  f->Lx = malloc((f->Lp[n] + 1) * sizeof(double));
  f->D = malloc((size_t)n * sizeof(double));
  double* Y = calloc(n, sizeof(double));
  uint32_t* pattern = malloc((size_t)n * sizeof(uint32_t));
  int rc = 0;
  for (uint32_t k = 0; k < n; ++k) {
    Y[k] = 0.0;
    uint32_t top = n;
    flag[k] = (int32_t)k;
    lnz[k] = 0;
    const uint32_t ko = f->perm[k];
    for (uint32_t p = M->rp[ko]; p < M->rp[ko + 1]; ++p) {
      uint32_t i = f->pinv[M->ci[p]];
      if (i > k) continue;
      Y[i] += M->v[p];
      uint32_t len = 0;
      for (; flag[i] != (int32_t)k; i = (uint32_t)parent[i]) {
        pattern[len++] = i;
        flag[i] = (int32_t)k;
      }
      while (len > 0) pattern[--top] = pattern[--len];
    }
    f->D[k] = Y[k];
    Y[k] = 0.0;
    for (; top < n; ++top) {
      const uint32_t i = pattern[top];
      const double yi = Y[i];
      Y[i] = 0.0;
      const size_t p2 = f->Lp[i] + lnz[i];
      for (size_t p = f->Lp[i]; p < p2; ++p) Y[f->Li[p]] -= f->Lx[p] * yi;
      const double l_ki = yi / f->D[i];
      f->D[k] -= l_ki * yi;
      f->Li[p2] = k;
      f->Lx[p2] = l_ki;
      lnz[i]++;
    }
    if (f->D[k] == 0.0) {
      rc = ORC_E_NUMERICAL; /* SingularSystem, solver.cpp:84-86 */
      break;
    }
  }
  free(parent);
  free(flag);
  free(lnz);
  free(Y);
  free(pattern);
  return rc;
}

/* Solves (P M P^T)(P x) = P b for a block of nb right-hand sides stored
 * interleaved (n x nb, row-major) in B (already permuted). */
static void ldl_solve_block(const ldl_factor* f, double* B, uint32_t nb) {
  const uint32_t n = f->n;
  for (uint32_t j = 0; j < n; ++j) {
    const double* bj = B + (size_t)j * nb;
    for (size_t p = f->Lp[j]; p < f->Lp[j + 1]; ++p) {
      double* bi = B + (size_t)f->Li[p] * nb;
      const double l = f->Lx[p];
      for (uint32_t c = 0; c < nb; ++c) bi[c] -= l * bj[c];
    }
  }
  for (uint32_t j = 0; j < n; ++j) {
    double* bj = B + (size_t)j * nb;
    const double d = f->D[j];
    for (uint32_t c = 0; c < nb; ++c) bj[c] /= d;
  }
  for (int64_t j = (int64_t)n - 1; j >= 0; --j) {
    double* bj = B + (size_t)j * nb;
    for (size_t p = f->Lp[j]; p < f->Lp[j + 1]; ++p) {
      const double* bi = B + (size_t)f->Li[p] * nb;
      const double l = f->Lx[p];
      for (uint32_t c = 0; c < nb; ++c) bj[c] -= l * bi[c];
    }
  }
}

/* x (n x W) = M^{-1} rhs (n x W), columns in chunks of 8 across threads. */
static void ldl_solve_multi(const ldl_factor* f, const double* rhs, double* x, uint32_t W,
                            int nthreads) {
  const uint32_t n = f->n;
  const uint32_t CH = 8;
  const uint32_t nchunks = (W + CH - 1) / CH;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
#endif
  for (uint32_t ch = 0; ch < nchunks; ++ch) {
    const uint32_t c0 = ch * CH, nb = (W - c0) < CH ? (W - c0) : CH;
    double* B = malloc((size_t)n * nb * sizeof(double));
    for (uint32_t k = 0; k < n; ++k) {
      const double* src = rhs + (size_t)f->perm[k] * W + c0;
      for (uint32_t c = 0; c < nb; ++c) B[(size_t)k * nb + c] = src[c];
    }
    ldl_solve_block(f, B, nb);
    for (uint32_t k = 0; k < n; ++k) {
      double* dst = x + (size_t)f->perm[k] * W + c0;
      for (uint32_t c = 0; c < nb; ++c) dst[c] = B[(size_t)k * nb + c];
    }
    free(B);
  }
  (void)nthreads;
}

/* y (n x W) = L x (n x W); L symmetric, so also L^T x.  Row sums in
 * ascending column order. */
static void spmm(uint32_t n, const uint32_t* lrow, const uint32_t* lcol, const double* lval,
                 const double* x, double* y, uint32_t W, int nthreads) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
  for (uint32_t i = 0; i < n; ++i) {
    double* o = y + (size_t)i * W;
    for (uint32_t c = 0; c < W; ++c) o[c] = 0.0;
    for (uint32_t p = lrow[i]; p < lrow[i + 1]; ++p) {
      const double v = lval[p];
      const double* xr = x + (size_t)lcol[p] * W;
      for (uint32_t c = 0; c < W; ++c) o[c] = o[c] + v * xr[c];
    }
  }
  (void)nthreads;
}

static size_t g_last_lnz = 0;
static double g_last_flops = 0.0;
/* Factor statistics of the last orc_solve_anchored call (test / docs aid). */
void orc_last_factor_stats(size_t* lnz, double* flops) {
  *lnz = g_last_lnz;
  *flops = g_last_flops;
}

int orc_solve_anchored(uint32_t n, const uint32_t* lrow, const uint32_t* lcol, const double* lval,
                       uint32_t W, const double* delta, uint32_t n_c, const uint32_t* idx,
                       const double* anchors, double* X, int nthreads) {
  if (n_c == 0) return ORC_E_CONFIG;
  for (uint32_t a = 0; a < n_c; ++a)
    if (idx[a] >= n) return ORC_E_INDEX;
  csr M = normal_matrix(n, lrow, lcol, lval, n_c, idx);
  ldl_factor f;
  f.n = n;
  f.perm = malloc((size_t)n * sizeof(uint32_t));
  f.pinv = malloc((size_t)n * sizeof(uint32_t));
  {
    nd_state st;
    st.M = &M;
    st.part = calloc(n, sizeof(int32_t));
    st.level = malloc((size_t)n * sizeof(int32_t));
    st.queue = malloc((size_t)n * sizeof(uint32_t));
    st.perm = f.perm;
    st.nperm = 0;
    st.next_id = 1;
    uint32_t* all = malloc((size_t)n * sizeof(uint32_t));
    for (uint32_t i = 0; i < n; ++i) all[i] = i;
    nd_recurse(&st, all, n, 0);
    free(all);
    free(st.part);
    free(st.level);
    free(st.queue);
    for (uint32_t k = 0; k < n; ++k) f.pinv[f.perm[k]] = k;
  }
  int rc = ldl_factorize(&M, &f);
  if (rc == 0) {
    g_last_lnz = f.Lp[n];
    double fl = 0.0;
    for (uint32_t j = 0; j < n; ++j) {
      const double c = (double)(f.Lp[j + 1] - f.Lp[j]);
      fl += c * c;
    }
    g_last_flops = fl;
    /* rhs = L^T delta + S^T a (solver.cpp:77-80) */
    double* rhs = malloc((size_t)n * W * sizeof(double));
    spmm(n, lrow, lcol, lval, delta, rhs, W, nthreads);
    for (uint32_t a = 0; a < n_c; ++a)
      for (uint32_t c = 0; c < W; ++c)
        rhs[(size_t)idx[a] * W + c] += anchors[(size_t)a * W + c];
    ldl_solve_multi(&f, rhs, X, W, nthreads);
    /* refine_anchored (solver.cpp:43-58) */
    double* lx = malloc((size_t)n * W * sizeof(double));
    spmm(n, lrow, lcol, lval, X, lx, W, nthreads);
    for (size_t t = 0; t < (size_t)n * W; ++t) lx[t] = delta[t] - lx[t];
    spmm(n, lrow, lcol, lval, lx, rhs, W, nthreads);
    for (uint32_t a = 0; a < n_c; ++a)
      for (uint32_t c = 0; c < W; ++c)
        rhs[(size_t)idx[a] * W + c] += anchors[(size_t)a * W + c] - X[(size_t)idx[a] * W + c];
    ldl_solve_multi(&f, rhs, lx, W, nthreads);
    for (size_t t = 0; t < (size_t)n * W; ++t) X[t] += lx[t];
    free(rhs);
    free(lx);
  }
  csr_free(&M);
  free(f.perm);
  free(f.pinv);
  if (rc == 0) {
    free(f.Lp);
    free(f.Li);
    free(f.Lx);
    free(f.D);
  }
  return rc;
}

/* Nested-dissection ordering + sparse LDL^T of an SPD CSR matrix (the
 * SimplicialLDLT stand-in shared by both solvers).  0 on success. */
static int ldl_build(csr* M, ldl_factor* f) {
  const uint32_t n = M->n;
  f->n = n;
  f->perm = malloc((size_t)n * sizeof(uint32_t));
  f->pinv = malloc((size_t)n * sizeof(uint32_t));
  nd_state st;
  st.M = M;
  st.part = calloc(n, sizeof(int32_t));
  st.level = malloc((size_t)n * sizeof(int32_t));
  st.queue = malloc((size_t)n * sizeof(uint32_t));
  st.perm = f->perm;
  st.nperm = 0;
  st.next_id = 1;
  uint32_t* all = malloc((size_t)n * sizeof(uint32_t));
  for (uint32_t i = 0; i < n; ++i) all[i] = i;
  nd_recurse(&st, all, n, 0);
  free(all);
  free(st.part);
  free(st.level);
  free(st.queue);
  for (uint32_t k = 0; k < n; ++k) f->pinv[f->perm[k]] = k;
  return ldl_factorize(M, f);
}

static void ldl_release(ldl_factor* f, int factored) {
  free(f->perm);
  free(f->pinv);
  if (factored) {
    free(f->Lp);
    free(f->Li);
    free(f->Lx);
    free(f->D);
  }
}

int orc_solve_mean_constrained(uint32_t n, const uint32_t* lrow, const uint32_t* lcol,
                               const double* lval, uint32_t W, const double* delta,
                               const double* means, double* X, int nthreads) {
  if (n < 2) return ORC_E_CONFIG;
  /* reduced = L[:, 1:]; normal = reduced^T reduced = (L^T L)[1:, 1:] (solver.cpp:116-117) */
  csr M = normal_matrix(n, lrow, lcol, lval, 0, NULL);
  csr Rm;
  Rm.n = n - 1;
  Rm.rp = malloc((size_t)n * sizeof(uint32_t));
  Rm.ci = malloc((size_t)M.rp[n] * sizeof(uint32_t));
  Rm.v = malloc((size_t)M.rp[n] * sizeof(double));
  uint32_t q = 0;
  Rm.rp[0] = 0;
  for (uint32_t i = 1; i < n; ++i) {
    for (uint32_t p = M.rp[i]; p < M.rp[i + 1]; ++p)
      if (M.ci[p] > 0) {
        Rm.ci[q] = M.ci[p] - 1;
        Rm.v[q++] = M.v[p];
      }
    Rm.rp[i] = q;
  }
  csr_free(&M);
  ldl_factor f;
  int rc = ldl_build(&Rm, &f);
  if (rc == 0) {
    const size_t nW = (size_t)n * W, mW = (size_t)(n - 1) * W;
    double* full = malloc(nW * sizeof(double));
    double* rhs = malloc(nW * sizeof(double));
    double* z = malloc(mW * sizeof(double));
    double* dz = malloc(mW * sizeof(double));
    /* z = solve(reduced^T delta); reduced^T = rows 1.. of L^T = L (solver.cpp:124) */
    spmm(n, lrow, lcol, lval, delta, rhs, W, nthreads);
    ldl_solve_multi(&f, rhs + W, z, W, nthreads);
    /* z += solve(reduced^T (delta - reduced z)); reduced z = L [0; z] (solver.cpp:125) */
    for (uint32_t c = 0; c < W; ++c) full[c] = 0.0;
    memcpy(full + W, z, mW * sizeof(double));
    spmm(n, lrow, lcol, lval, full, rhs, W, nthreads);
    for (size_t t = 0; t < nW; ++t) full[t] = delta[t] - rhs[t];
    spmm(n, lrow, lcol, lval, full, rhs, W, nthreads);
    ldl_solve_multi(&f, rhs + W, dz, W, nthreads);
    for (size_t t = 0; t < mW; ++t) z[t] += dz[t];
    /* x = [0; z], each column shifted to its mean (solver.cpp:126-131) */
    for (uint32_t c = 0; c < W; ++c) X[c] = 0.0;
    memcpy(X + W, z, mW * sizeof(double));
    for (uint32_t c = 0; c < W; ++c) {
      double sum = 0.0;
      for (uint32_t i = 0; i < n; ++i) sum += X[(size_t)i * W + c];
      const double shift = means[c] - sum / (double)n;
      for (uint32_t i = 0; i < n; ++i) X[(size_t)i * W + c] += shift;
    }
    free(full);
    free(rhs);
    free(z);
    free(dz);
  }
  csr_free(&Rm);
  ldl_release(&f, rc == 0);
  return rc;
}

/* ======================================================================== */
/* encode / decode (src/codec.cpp:351-552)                                   */
/* ======================================================================== */

int orc_encode(uint32_t n, uint32_t F, const double* const axes[3], const uint32_t* faces,
               uint32_t n_faces, uint32_t k_l, const int* row_bits, double anchor_fraction,
               int anchor_bits, int dict_bits, int rounds, uint64_t basis_seed, orc_encoded* out,
               double* U_out, double* evals_out, orc_timing* tm, int nthreads) {
  return orc_encode_variant(4, n, F, axes, faces, n_faces, k_l, row_bits, anchor_fraction,
                            anchor_bits, dict_bits, rounds, basis_seed, out, U_out, evals_out, tm,
                            nthreads);
}

static int uses_anchors(int v) { return v == 3 || v == 4 || v == 5; }  /* stream.hpp:77-79 */
static int uses_means(int v) { return v == 0 || v == 1; }    /* stream.hpp:80-82 */

int orc_encode_variant(int variant, uint32_t n, uint32_t F, const double* const axes[3],
                       const uint32_t* faces, uint32_t n_faces, uint32_t k_l, const int* row_bits,
                       double anchor_fraction, int anchor_bits, int dict_bits, int rounds,
                       uint64_t basis_seed, orc_encoded* out, double* U_out, double* evals_out,
                       orc_timing* tm, int nthreads) {
  if (variant < 0 || variant > 4) return ORC_E_CONFIG;
  orc_timing dummy;
  if (!tm) tm = &dummy;
  memset(tm, 0, sizeof(*tm));
  double t0 = now_s();
  /* validate_sequence + check_config (codec.cpp:352-363, 69-120) */
  if (orc_validate(n, F, faces, n_faces, axes[0], axes[1], axes[2])) return ORC_E_INDEX;
  if (k_l > F) return ORC_E_CONFIG;
  if (anchor_fraction < 0.0 || anchor_fraction > 1.0) return ORC_E_CONFIG;
  if (anchor_bits < 1 || anchor_bits > 16 || dict_bits < 1 || dict_bits > 16) return ORC_E_CONFIG;
  for (uint32_t r = 0; r < k_l; ++r)
    if (row_bits[r] < 1 || row_bits[r] > 16) return ORC_E_CONFIG;
  out->n = n;
  out->F = F;
  out->k_l = k_l;
  out->variant = variant;
  out->n_c = uses_anchors(variant) ? orc_anchor_count(n, anchor_fraction) : 0;
  out->n_faces = n_faces;
  out->faces = faces;
  out->anchor_bits = anchor_bits;
  out->dict_bits = dict_bits;
  if (out->diff_bits == 0) out->diff_bits = 8;
  uint32_t* arp = malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* acol = malloc((size_t)6 * n_faces * sizeof(uint32_t));
  long nnz = orc_build_connectivity(faces, n_faces, n, arp, acol);
  uint32_t* lrow = malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* lcol = malloc(((size_t)n + nnz) * sizeof(uint32_t));
  double* lval = malloc(((size_t)n + nnz) * sizeof(double));
  orc_build_laplacian(n, arp, acol, 0, lrow, lcol, lval);
  tm->t_connectivity = now_s() - t0;

  int rc = 0;
  double* R = malloc((size_t)F * F * sizeof(double));
  double* U = malloc((size_t)F * F * sizeof(double));
  double* ev = malloc((size_t)F * sizeof(double));
  double* delta = malloc((size_t)n * F * sizeof(double));
  double* C = malloc((size_t)(k_l ? k_l : 1) * n * sizeof(double));
  for (int a = 0; a < 3 && !rc; ++a) {
    const double* X = axes[a];
    t0 = now_s();
    orc_autocorrelation(n, F, X, R);
    tm->t_gram += now_s() - t0;
    t0 = now_s();
    rc = orc_basis(F, k_l, R, rounds, basis_seed + (uint64_t)a, U, ev);
    tm->t_eigen += now_s() - t0;
    if (rc) break;
    if (U_out) memcpy(U_out + (size_t)a * F * F, U, (size_t)F * F * sizeof(double));
    if (evals_out) memcpy(evals_out + (size_t)a * F, ev, (size_t)F * sizeof(double));
    /* encode_dictionaries first block: pack_matrix over [-1, 1] (codec.cpp:122-129,300-301) */
    for (size_t t = 0; t < (size_t)F * F; ++t)
      out->dict_q[a][t] = orc_quantize(-1.0f, 1.0f, dict_bits, U[t]);
    t0 = now_s();
    if (variant == 2)  /* v2v: the trajectories themselves (codec.cpp:416-417) */
      memcpy(delta, X, (size_t)n * F * sizeof(double));
    else
      orc_delta(n, F, lrow, lcol, lval, X, delta);
    tm->t_delta += now_s() - t0;
    if (uses_means(variant))  /* traj.row(f).mean() as float (codec.cpp:432-441) */
      for (uint32_t f = 0; f < F; ++f) {
        double sum = 0.0;
        for (uint32_t i = 0; i < n; ++i) sum += X[(size_t)i * F + f];
        out->means[a][f] = (float)(sum / (double)n);
      }
    /* coeffs = U^T delta^T, rows r < k_l (codec.cpp:420) */
    t0 = now_s();
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (uint32_t i = 0; i < n; ++i) {
      const double* d = delta + (size_t)i * F;
      for (uint32_t r = 0; r < k_l; ++r) {
        const double* u = U + (size_t)r * F;
        double s = 0.0;
        for (uint32_t f = 0; f < F; ++f) s = s + u[f] * d[f];
        C[(size_t)r * n + i] = s;
      }
    }
    tm->t_project += now_s() - t0;
    t0 = now_s();
    orc_quantize_rows(k_l, n, C, row_bits, out->row_min[a], out->row_max[a], out->coeff_q[a]);
    for (uint32_t r = 0; r < k_l; ++r) out->row_bits[a][r] = (uint8_t)row_bits[r];
    tm->t_quantize += now_s() - t0;
  }
  /* anchors (codec.cpp:444-471) */
  t0 = now_s();
  if (!rc && out->n_c) rc = orc_select_anchors(n, out->n_c, 0, 0, out->anchor_idx);
  for (int a = 0; a < 3 && !rc && out->n_c; ++a) {
    const double* X = axes[a];
    double lo = INFINITY, hi = -INFINITY;
    for (uint32_t t = 0; t < out->n_c; ++t) {
      const double* x = X + (size_t)out->anchor_idx[t] * F;
      double cmin = x[0], cmax = x[0];
      for (uint32_t f = 1; f < F; ++f) {
        if (x[f] < cmin) cmin = x[f];
        if (x[f] > cmax) cmax = x[f];
      }
      lo = lo < cmin ? lo : cmin;
      hi = hi > cmax ? hi : cmax;
    }
    float flo, fhi;
    orc_widened_range(lo, hi, &flo, &fhi);
    out->anchor_min[a] = flo;
    out->anchor_max[a] = fhi;
    for (uint32_t t = 0; t < out->n_c; ++t) {
      const double* x = X + (size_t)out->anchor_idx[t] * F;
      for (uint32_t f = 0; f < F; ++f)
        out->anchor_q[a][(size_t)t * F + f] = orc_quantize(flo, fhi, anchor_bits, x[f]);
    }
  }
  tm->t_anchors = now_s() - t0;
  free(arp);
  free(acol);
  free(lrow);
  free(lcol);
  free(lval);
  free(R);
  free(U);
  free(ev);
  free(delta);
  free(C);
  return rc;
}

/* ======================================================================== */
/* blocks variant (n_b > 1)                                                   */
/* ======================================================================== */

static uint32_t nb_of(const orc_encoded* e) { return e->n_b ? e->n_b : 1; }

/* align_signs (src/spectral.cpp:122-131): flip columns with prev . cur < 0. */
static void align_signs(uint32_t m, const double* prev, double* U) {
  for (uint32_t j = 0; j < m; ++j) {
    const double* p = prev + (size_t)j * m;
    double* u = U + (size_t)j * m;
    double d = 0.0;
    for (uint32_t i = 0; i < m; ++i) d += p[i] * u[i];
    if (d < 0.0)
      for (uint32_t i = 0; i < m; ++i) u[i] = -u[i];
  }
}

/* k_f x k_f autocorrelation of frames [f0, f0 + kf) of the padded n x Fp
 * trajectory (spectral.cpp:35-39 on a.middleRows(b * k_f, k_f)). */
static void block_autocorrelation(uint32_t n, uint32_t Fp, uint32_t f0, uint32_t kf,
                                  const double* Xp, double* R) {
  for (uint32_t g = 0; g < kf; ++g)
    for (uint32_t f = 0; f < kf; ++f) {
      double s = 0.0;
      for (uint32_t i = 0; i < n; ++i) s += Xp[(size_t)i * Fp + f0 + f] * Xp[(size_t)i * Fp + f0 + g];
      R[(size_t)g * kf + f] = s;
    }
  for (uint32_t g = 0; g < kf; ++g)
    for (uint32_t f = 0; f < g; ++f) {
      const double s = 0.5 * (R[(size_t)g * kf + f] + R[(size_t)f * kf + g]);
      R[(size_t)g * kf + f] = s;
      R[(size_t)f * kf + g] = s;
    }
}

int orc_encode_blocks(uint32_t n, uint32_t F, const double* const axes[3], const uint32_t* faces,
                      uint32_t n_faces, uint32_t n_b, uint32_t k_l, const int* row_bits,
                      double anchor_fraction, int anchor_bits, int dict_bits, int diff_bits,
                      int t_max, double stop_tol, orc_encoded* out, double* U_out, int nthreads) {
  /* validate_sequence + check_config (codec.cpp:352-363, 69-120) */
  if (orc_validate(n, F, faces, n_faces, axes[0], axes[1], axes[2])) return ORC_E_INDEX;
  if (n_b < 1 || n_b > F || t_max < 1) return ORC_E_CONFIG;
  if (anchor_fraction < 0.0 || anchor_fraction > 1.0) return ORC_E_CONFIG;
  if (anchor_bits < 1 || anchor_bits > 16 || dict_bits < 1 || dict_bits > 16 || diff_bits < 1 ||
      diff_bits > 16)
    return ORC_E_CONFIG;
  const uint32_t pad = (n_b - F % n_b) % n_b, Fp = F + pad, kf = Fp / n_b;
  if (k_l > kf) return ORC_E_CONFIG;
  for (uint32_t r = 0; r < k_l; ++r)
    if (row_bits[r] < 1 || row_bits[r] > 16) return ORC_E_CONFIG;
  out->n = n;
  out->F = F;
  out->k_l = k_l;
  out->variant = 5;
  out->n_b = n_b;
  out->pad = pad;
  out->n_c = orc_anchor_count(n, anchor_fraction);
  out->n_faces = n_faces;
  out->faces = faces;
  out->anchor_bits = anchor_bits;
  out->dict_bits = dict_bits;
  out->diff_bits = diff_bits;
  uint32_t* arp = malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* acol = malloc((size_t)6 * n_faces * sizeof(uint32_t));
  long nnz = orc_build_connectivity(faces, n_faces, n, arp, acol);
  uint32_t* lrow = malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* lcol = malloc(((size_t)n + nnz) * sizeof(uint32_t));
  double* lval = malloc(((size_t)n + nnz) * sizeof(double));
  orc_build_laplacian(n, arp, acol, 0, lrow, lcol, lval);

  const size_t kk = (size_t)kf * kf;
  double* Xp = malloc((size_t)n * Fp * sizeof(double));
  double* delta = malloc((size_t)n * Fp * sizeof(double));
  double* R = malloc(kk * sizeof(double));
  double* D = malloc(n_b * kk * sizeof(double));    /* dicts[b] */
  double* Dec = malloc(kk * sizeof(double));        /* payload.decoded.back() */
  double* cur = malloc(kk * sizeof(double));
  double* C = malloc((size_t)(k_l ? k_l : 1) * n * sizeof(double));
  int rc = 0;
  for (int a = 0; a < 3 && !rc; ++a) {
    /* pad_frames (codec.cpp:43-49): repeat the last frame */
    for (uint32_t i = 0; i < n; ++i) {
      memcpy(Xp + (size_t)i * Fp, axes[a] + (size_t)i * F, (size_t)F * sizeof(double));
      for (uint32_t p = 0; p < pad; ++p) Xp[(size_t)i * Fp + F + p] = axes[a][(size_t)i * F + F - 1];
    }
    /* block_dictionaries (codec.cpp:149-172) */
    for (uint32_t b = 0; b < n_b && !rc; ++b) {
      double* U = D + b * kk;
      block_autocorrelation(n, Fp, b * kf, kf, Xp, R);
      if (b == 0) {
        rc = orc_full_eigenbasis(kf, R, U, NULL);
      } else {
        if (orc_orthogonal_iterations(kf, R, D + (b - 1) * kk, t_max, stop_tol, U))
          rc = orc_full_eigenbasis(kf, R, U, NULL);  /* catch (RankDeficiency) */
        if (!rc) align_signs(kf, D + (b - 1) * kk, U);
      }
    }
    if (rc) break;
    if (U_out) memcpy(U_out + (size_t)a * n_b * kk, D, n_b * kk * sizeof(double));
    /* encode_dictionaries (codec.cpp:290-328), auto_realign = true */
    uint32_t* dq = out->dict_q[a];
    for (size_t t = 0; t < kk; ++t) {
      dq[t] = orc_quantize(-1.0f, 1.0f, dict_bits, D[t]);
      Dec[t] = orc_dequantize(-1.0f, 1.0f, dict_bits, dq[t]);
    }
    for (uint32_t b = 1; b < n_b; ++b) {
      memcpy(cur, D + b * kk, kk * sizeof(double));
      for (uint32_t j = 0; j < kf; ++j) {
        double* c = cur + (size_t)j * kf;
        const double* p = Dec + (size_t)j * kf;
        double straight = 0.0, flipped = 0.0;
        for (uint32_t i = 0; i < kf; ++i) {
          const double d = c[i] - p[i], e = -c[i] - p[i];
          straight += d * d;
          flipped += e * e;
        }
        if (straight > 2.0 && flipped < straight)
          for (uint32_t i = 0; i < kf; ++i) c[i] = -c[i];
      }
      double lo = INFINITY, hi = -INFINITY;
      for (size_t t = 0; t < kk; ++t) {
        cur[t] = cur[t] - Dec[t];  /* diff = cur - prev */
        if (cur[t] < lo) lo = cur[t];
        if (cur[t] > hi) hi = cur[t];
      }
      float flo, fhi;
      orc_widened_range(lo, hi, &flo, &fhi);
      out->diff_min[a][b - 1] = flo;
      out->diff_max[a][b - 1] = fhi;
      uint32_t* q = dq + b * kk;
      for (size_t t = 0; t < kk; ++t) {
        q[t] = orc_quantize(flo, fhi, diff_bits, cur[t]);
        Dec[t] = Dec[t] + orc_dequantize(flo, fhi, diff_bits, q[t]);
      }
    }
    /* per block: delta_b = L * block_traj^T, coeffs = dicts[b]^T delta_b^T
     * (codec.cpp:411-429); delta is column-separable, so delta of the
     * padded trajectory restricted to the block's frames. */
    orc_delta(n, Fp, lrow, lcol, lval, Xp, delta);
    for (uint32_t b = 0; b < n_b; ++b) {
      const double* U = D + b * kk;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
      for (uint32_t i = 0; i < n; ++i) {
        const double* d = delta + (size_t)i * Fp + (size_t)b * kf;
        for (uint32_t r = 0; r < k_l; ++r) {
          const double* u = U + (size_t)r * kf;
          double s = 0.0;
          for (uint32_t f = 0; f < kf; ++f) s = s + u[f] * d[f];
          C[(size_t)r * n + i] = s;
        }
      }
      const size_t ro = (size_t)b * k_l;
      orc_quantize_rows(k_l, n, C, row_bits, out->row_min[a] + ro, out->row_max[a] + ro,
                        out->coeff_q[a] + ro * n);
      for (uint32_t r = 0; r < k_l; ++r) out->row_bits[a][ro + r] = (uint8_t)row_bits[r];
    }
  }
  /* anchors on the unpadded trajectories (codec.cpp:444-471) */
  if (!rc) rc = orc_select_anchors(n, out->n_c, 0, 0, out->anchor_idx);
  for (int a = 0; a < 3 && !rc; ++a) {
    const double* X = axes[a];
    double lo = INFINITY, hi = -INFINITY;
    for (uint32_t t = 0; t < out->n_c; ++t)
      for (uint32_t f = 0; f < F; ++f) {
        const double v = X[(size_t)out->anchor_idx[t] * F + f];
        if (v < lo) lo = v;
        if (v > hi) hi = v;
      }
    float flo, fhi;
    orc_widened_range(lo, hi, &flo, &fhi);
    out->anchor_min[a] = flo;
    out->anchor_max[a] = fhi;
    for (uint32_t t = 0; t < out->n_c; ++t)
      for (uint32_t f = 0; f < F; ++f)
        out->anchor_q[a][(size_t)t * F + f] =
            orc_quantize(flo, fhi, anchor_bits, X[(size_t)out->anchor_idx[t] * F + f]);
  }
  free(arp);
  free(acol);
  free(lrow);
  free(lcol);
  free(lval);
  free(Xp);
  free(delta);
  free(R);
  free(D);
  free(Dec);
  free(cur);
  free(C);
  return rc;
}

/* decode_dictionaries (codec.cpp:330-349) */
int orc_decode_dictionaries(const orc_encoded* in, int a, double* out) {
  const uint32_t n_b = nb_of(in), kf = (in->F + in->pad) / n_b;
  const size_t kk = (size_t)kf * kf;
  const uint32_t dlev = 1u << in->dict_bits, flev = 1u << in->diff_bits;
  int rc = 0;
  for (size_t t = 0; t < kk; ++t) {
    if (in->dict_q[a][t] >= dlev) rc = ORC_E_CORRUPT;
    out[t] = orc_dequantize(-1.0f, 1.0f, in->dict_bits, in->dict_q[a][t]);
  }
  for (uint32_t b = 1; b < n_b; ++b) {
    const float mn = in->diff_min[a][b - 1], mx = in->diff_max[a][b - 1];
    const uint32_t* q = in->dict_q[a] + b * kk;
    for (size_t t = 0; t < kk; ++t) {
      if (q[t] >= flev) rc = ORC_E_CORRUPT;
      out[b * kk + t] = out[(b - 1) * kk + t] + orc_dequantize(mn, mx, in->diff_bits, q[t]);
    }
  }
  return rc;
}

int orc_decode(const orc_encoded* in, double* const axes_out[3], orc_timing* tm, int nthreads) {
  orc_timing dummy;
  if (!tm) tm = &dummy;
  memset(tm, 0, sizeof(*tm));
  const uint32_t n = in->n, F = in->F, k_l = in->k_l, n_c = in->n_c;
  /* blocks (n_b > 1): the solve runs over the F + pad padded frames
   * (codec.cpp:483-495, 527-549), blocks of k_f frames */
  const uint32_t nb = nb_of(in), Fp = F + (nb > 1 ? in->pad : 0), kf = Fp / nb;
  const uint32_t W = 3 * Fp;
  double t0 = now_s();
  uint32_t* arp = malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* acol = malloc((size_t)6 * in->n_faces * sizeof(uint32_t));
  long nnz = orc_build_connectivity(in->faces, in->n_faces, n, arp, acol);
  if (nnz < 0) {
    free(arp);
    free(acol);
    return (int)-nnz;
  }
  uint32_t* lrow = malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* lcol = malloc(((size_t)n + nnz) * sizeof(uint32_t));
  double* lval = malloc(((size_t)n + nnz) * sizeof(double));
  orc_build_laplacian(n, arp, acol, 0, lrow, lcol, lval);
  tm->t_connectivity = now_s() - t0;
  int rc = 0;
  double* delta = malloc((size_t)n * W * sizeof(double)); /* n x 3F */
  double* anchors = malloc((size_t)n_c * W * sizeof(double));
  double* Ut = malloc((size_t)nb * kf * kf * sizeof(double));
  double* Cq = malloc((size_t)(k_l ? k_l : 1) * n * sizeof(double));
  for (int a = 0; a < 3 && !rc; ++a) {
    /* anchor_matrix (codec.cpp:174-195) */
    const uint32_t alev = 1u << in->anchor_bits;
    for (uint32_t t = 0; t < n_c; ++t)
      for (uint32_t f = 0; f < F; ++f) {
        const uint32_t lv = in->anchor_q[a][(size_t)t * F + f];
        if (lv >= alev) rc = ORC_E_CORRUPT;
        anchors[(size_t)t * W + (size_t)a * Fp + f] =
            orc_dequantize(in->anchor_min[a], in->anchor_max[a], in->anchor_bits, lv);
      }
    for (uint32_t t = 0; t < n_c; ++t)  /* padded columns repeat the last frame */
      for (uint32_t f = F; f < Fp; ++f)
        anchors[(size_t)t * W + (size_t)a * Fp + f] = anchors[(size_t)t * W + (size_t)a * Fp + F - 1];
    /* decode_dictionaries / unpack_matrix (codec.cpp:330-349,131-142) */
    t0 = now_s();
    if (orc_decode_dictionaries(in, a, Ut)) rc = ORC_E_CORRUPT;
    tm->t_dict_decode += now_s() - t0;
    if (rc) break;
    /* dequantize_rows + delta~ = (U~ coeffs)^T (codec.cpp:528-533) */
    t0 = now_s();
    for (uint32_t b = 0; b < nb && !rc; ++b) {
      const size_t ro = (size_t)b * k_l;
      rc = orc_dequantize_rows(k_l, k_l, n, in->row_min[a] + ro, in->row_max[a] + ro,
                               in->row_bits[a] + ro, in->coeff_q[a] + ro * n, Cq);
      if (rc) break;
      const double* Ub = Ut + (size_t)b * kf * kf;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
      for (uint32_t i = 0; i < n; ++i) {
        double* o = delta + (size_t)i * W + (size_t)a * Fp + (size_t)b * kf;
        for (uint32_t f = 0; f < kf; ++f) o[f] = 0.0;
        for (uint32_t r = 0; r < k_l; ++r) {
          const double c = Cq[(size_t)r * n + i];
          const double* u = Ub + (size_t)r * kf;
          for (uint32_t f = 0; f < kf; ++f) o[f] = o[f] + u[f] * c;
        }
      }
    }
    if (rc) break;
    tm->t_reconstruct += now_s() - t0;
  }
  if (!rc) {
    /* solve_anchored, Parallel (codec.cpp:537-539): the reference factors M
     * once per axis; M does not depend on the axis, so all 3F columns are
     * solved against one factorisation here.  pca_qs (Serial) refactors per
     * column (solver.cpp:92-100): the same factor and column-separable solves.
     * v2v needs no solve (codec.cpp:520-524); pca / pca_q the mean-
     * constrained one (codec.cpp:540-546). */
    t0 = now_s();
    double* X = malloc((size_t)n * W * sizeof(double));
    if (in->variant == 2) {
      memcpy(X, delta, (size_t)n * W * sizeof(double));
    } else if (uses_means(in->variant)) {
      double* mw = malloc((size_t)W * sizeof(double));
      for (int a = 0; a < 3; ++a)
        for (uint32_t f = 0; f < F; ++f) mw[(size_t)a * F + f] = (double)in->means[a][f];
      rc = orc_solve_mean_constrained(n, lrow, lcol, lval, W, delta, mw, X, nthreads);
      free(mw);
    } else {
      rc = orc_solve_anchored(n, lrow, lcol, lval, W, delta, n_c, in->anchor_idx, anchors, X,
                              nthreads);
    }
    for (int a = 0; a < 3 && !rc; ++a)
      for (uint32_t i = 0; i < n; ++i)
        memcpy(axes_out[a] + (size_t)i * F, X + (size_t)i * W + (size_t)a * Fp,
               (size_t)F * sizeof(double));
    free(X);
    tm->t_solve = now_s() - t0;
  }
  free(arp);
  free(acol);
  free(lrow);
  free(lcol);
  free(lval);
  free(delta);
  free(anchors);
  free(Ut);
  free(Cq);
  return rc;
}

/* ======================================================================== */
/* stream.cpp / metrics.cpp                                                  */
/* ======================================================================== */

/* BitWriter (src/quantize.cpp:50-69): MSB-first, zero-padded on take(). */
typedef struct {
  uint8_t* out; /* may be NULL (size query) */
  size_t pos;
  uint64_t acc;
  int fill;
} bitw;

static void bw_put(bitw* w, uint32_t v, int bits) {
  w->acc = (w->acc << bits) | (v & ((bits == 32) ? 0xFFFFFFFFu : ((1u << bits) - 1u)));
  w->fill += bits;
  while (w->fill >= 8) {
    w->fill -= 8;
    if (w->out) w->out[w->pos] = (uint8_t)(w->acc >> w->fill);
    w->pos++;
  }
}
static void bw_flush(bitw* w) {
  if (w->fill > 0) {
    if (w->out) w->out[w->pos] = (uint8_t)(w->acc << (8 - w->fill));
    w->pos++;
    w->fill = 0;
  }
  w->acc = 0;
}

static void put_u8(uint8_t* o, size_t* p, uint8_t v) {
  if (o) o[*p] = v;
  *p += 1;
}
static void put_u16(uint8_t* o, size_t* p, uint16_t v) {
  put_u8(o, p, (uint8_t)v);
  put_u8(o, p, (uint8_t)(v >> 8));
}
static void put_u32(uint8_t* o, size_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) put_u8(o, p, (uint8_t)(v >> (8 * i)));
}
static void put_f32(uint8_t* o, size_t* p, float v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  put_u32(o, p, u);
}

/* src/stream.cpp:172-292 for the quantised payloads of variants 0-5. */
size_t orc_serialize(const orc_encoded* e, uint8_t* o, orc_sections* s) {
  orc_sections sz;
  memset(&sz, 0, sizeof(sz));
  size_t p = 0;
  const char magic[4] = {'D', 'M', 'C', '1'};
  for (int i = 0; i < 4; ++i) put_u8(o, &p, (uint8_t)magic[i]);
  put_u16(o, &p, 1);  /* version */
  put_u8(o, &p, (uint8_t)e->variant);
  put_u8(o, &p, 0);   /* flags */
  put_u32(o, &p, e->n);
  put_u32(o, &p, e->F);
  const uint32_t nb = nb_of(e), kf = (e->F + (nb > 1 ? e->pad : 0)) / nb;
  put_u16(o, &p, (uint16_t)nb);
  put_u16(o, &p, (uint16_t)(nb > 1 ? e->pad : 0));
  put_u32(o, &p, e->k_l);
  put_u32(o, &p, e->n_c);
  put_u8(o, &p, (uint8_t)e->anchor_bits);
  put_u8(o, &p, (uint8_t)e->dict_bits);
  put_u8(o, &p, (uint8_t)(e->diff_bits ? e->diff_bits : 8));
  put_u8(o, &p, 0);
  sz.header = p;
  put_u32(o, &p, e->n_faces);
  for (size_t t = 0; t < 3 * (size_t)e->n_faces; ++t) put_u32(o, &p, e->faces[t]);
  sz.connectivity = p - sz.header;
  for (int a = 0; a < 3; ++a) {
    size_t start = p;
    const size_t kk = (size_t)kf * kf;
    bitw w = {o, p, 0, 0};
    for (size_t t = 0; t < kk; ++t) bw_put(&w, e->dict_q[a][t], e->dict_bits);
    bw_flush(&w);
    p = w.pos;
    sz.dict_payload += p - start;
    for (uint32_t b = 1; b < nb; ++b) {  /* dict_diffs (stream.cpp:218-227) */
      start = p;
      put_f32(o, &p, e->diff_min[a][b - 1]);
      put_f32(o, &p, e->diff_max[a][b - 1]);
      sz.dict_ranges += p - start;
      start = p;
      bitw d = {o, p, 0, 0};
      for (size_t t = 0; t < kk; ++t) bw_put(&d, e->dict_q[a][b * kk + t], e->diff_bits);
      bw_flush(&d);
      p = d.pos;
      sz.dict_payload += p - start;
    }
    for (uint32_t b = 0; b < nb; ++b) {  /* one CoeffBlock per block (stream.cpp:229-251) */
      const size_t ro = (size_t)b * e->k_l;
      start = p;
      for (uint32_t r = 0; r < e->k_l; ++r) {
        put_f32(o, &p, e->row_min[a][ro + r]);
        put_f32(o, &p, e->row_max[a][ro + r]);
        put_u8(o, &p, e->row_bits[a][ro + r]);
      }
      sz.coeff_headers += p - start;
      start = p;
      w.pos = p;
      w.acc = 0;
      w.fill = 0;
      for (uint32_t r = 0; r < e->k_l; ++r) {
        if (e->row_min[a][ro + r] == e->row_max[a][ro + r]) continue;
        const uint32_t* q = e->coeff_q[a] + (ro + r) * e->n;
        for (uint32_t i = 0; i < e->n; ++i) bw_put(&w, q[i], e->row_bits[a][ro + r]);
      }
      bw_flush(&w);
      p = w.pos;
      sz.coeff_payload += p - start;
    }
    if (uses_means(e->variant)) {  /* stream.cpp:255-263 */
      start = p;
      for (uint32_t f = 0; f < e->F; ++f) put_f32(o, &p, e->means[a][f]);
      sz.means += p - start;
    }
  }
  if (!uses_anchors(e->variant)) {
    if (s) *s = sz;
    return p;
  }
  size_t start = p;
  for (uint32_t t = 0; t < e->n_c; ++t) put_u32(o, &p, e->anchor_idx[t]);
  sz.anchor_indices = p - start;
  for (int a = 0; a < 3; ++a) {
    start = p;
    put_f32(o, &p, e->anchor_min[a]);
    put_f32(o, &p, e->anchor_max[a]);
    sz.anchor_ranges += p - start;
    start = p;
    bitw w = {o, p, 0, 0};
    for (size_t t = 0; t < (size_t)e->n_c * e->F; ++t) bw_put(&w, e->anchor_q[a][t], e->anchor_bits);
    bw_flush(&w);
    p = w.pos;
    sz.anchor_payload += p - start;
  }
  if (s) *s = sz;
  return p;
}

/* src/metrics.cpp:46-59 */
void orc_rate_exact(const orc_sections* s, uint32_t n, uint32_t F, double out[5]) {
  const double tv = (double)n * F;
  out[0] = 8.0 * s->coeff_payload / tv;
  out[1] = 8.0 * (s->anchor_indices + s->anchor_payload) / tv;
  out[2] = 8.0 * s->dict_payload / tv;
  out[3] = 8.0 *
           (s->header + s->connectivity + s->dict_ranges + s->coeff_headers + s->means +
            s->anchor_ranges) /
           tv;
  out[4] = out[0] + out[1] + out[2] + out[3];
}

/* src/metrics.cpp:67-79 */
void orc_frame_rms(uint32_t n, uint32_t F, const double* const a[3], const double* const b[3],
                   double* out) {
  for (uint32_t f = 0; f < F; ++f) {
    double sum = 0.0;
    for (int ax = 0; ax < 3; ++ax) {
      double s = 0.0;
      for (uint32_t i = 0; i < n; ++i) {
        const double d = a[ax][(size_t)i * F + f] - b[ax][(size_t)i * F + f];
        s += d * d;
      }
      sum += s;
    }
    out[f] = sqrt(sum / n);
  }
}
