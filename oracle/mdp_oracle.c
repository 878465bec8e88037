/*
 * mdp_oracle.c — C/OpenMP restatement of the reference iPI path.
 * TEST INFRASTRUCTURE ONLY: used by tests/ (parity at sizes the numpy oracle
 * cannot reach) and by bench.py's CPU legs (cpu_baseline, --impl reference).
 * Never linked into libipi_b200.so.
 *
 * Restates (paths relative to /root/reference/pkg/src/mdpsolve):
 *   spmv row sums     sparse.py:189-215 via np.add.reduceat (:126-139): the
 *                     row sum is a[0] + pairwise(a[1:]) with numpy's published
 *                     8-way-unrolled pairwise summation (numpy umath
 *                     loops_utils pairwise_sum, PW_BLOCKSIZE 128), so greedy /
 *                     spmv match the reference bitwise.
 *   greedy            bellman.py:44-68 (gamma*pv first, first-index argmin/argmax)
 *   gather            sparse.py:243-269
 *   apply             sparse.py:294-295 (x - gamma*(P x))
 *   richardson        inner.py:216-226
 *   gmres(30)         inner.py:229-292 (MGS, Givens, est_target tightening)
 *   inner_solve       inner.py:163-213 (floor 1e-14*max(1,||b||))
 *   solve             driver.py:109-209 (statuses, stall window 50)
 * Dots use fixed 4096-element blocks summed in block order, so results do not
 * depend on the thread count (np.dot/BLAS order is not reproducible; GMRES is
 * therefore validated to tolerance, not bitwise).
 *
 * Also: the C2/C5 locality generator (Philox4x32-10, same integer stream as
 * generators.py / gen.cu) so the CPU baseline builds its bounded sample fast.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define RESTART 30
#define DOT_BLOCK 4096

static void set_threads(int nt) {
#ifdef _OPENMP
  if (nt > 0) omp_set_num_threads(nt);
#else
  (void)nt;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* numpy pairwise summation of a contiguous run (loops_utils.h.src) */
static double pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, n2) + pairwise(a + n2, n - n2);
  }
}

/* one CSR row: prod = val*x[col] rounded, then reduceat's a[0] + pairwise(a[1:]) */
static double row_sum(const int64_t* rp, const int32_t* col, const double* val, const double* x,
                      int64_t r, double* scratch) {
  const int64_t p0 = rp[r], len = rp[r + 1] - rp[r];
  if (len == 0) return 0.0;
  for (int64_t i = 0; i < len; ++i) scratch[i] = val[p0 + i] * x[col[p0 + i]];
  return scratch[0] + pairwise(scratch + 1, len - 1);
}

static int64_t max_row_len(const int64_t* rp, int64_t rows) {
  int64_t mx = 0;
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t l = rp[r + 1] - rp[r];
    if (l > mx) mx = l;
  }
  return mx;
}

void orc_spmv(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
              const double* x, double* y, int nthreads) {
  set_threads(nthreads);
  const int64_t L = max_row_len(rp, rows) + 1;
#pragma omp parallel
  {
    double* scratch = (double*)malloc(sizeof(double) * L);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < rows; ++r) y[r] = row_sum(rp, col, val, x, r, scratch);
    free(scratch);
  }
}

/* greedy_policy over states [0, n_states) of the (n_states*m) row block;
 * v has n_cols entries (global V).  Returns max |v[state0+s] - applied[s]|. */
double orc_greedy(int64_t n_states, int32_t m, const int64_t* rp, const int32_t* col,
                  const double* val, const double* cost, double gamma, int maximize,
                  const double* v, int64_t state0, int64_t* pi, double* applied, int nthreads) {
  set_threads(nthreads);
  const int64_t L = max_row_len(rp, n_states * m) + 1;
  double res = 0.0;
#pragma omp parallel reduction(max : res)
  {
    double* scratch = (double*)malloc(sizeof(double) * L);
#pragma omp for schedule(static)
    for (int64_t s = 0; s < n_states; ++s) {
      int best = 0;
      double bq = 0.0;
      for (int a = 0; a < m; ++a) {
        const int64_t r = s * m + a;
        const double pv = row_sum(rp, col, val, v, r, scratch);
        const double q = cost[r] + gamma * pv;
        if (a == 0 || (maximize ? q > bq : q < bq)) {
          bq = q;
          best = a;
        }
      }
      pi[s] = best;
      applied[s] = bq;
      const double d = fabs(v[state0 + s] - bq);
      if (d > res) res = d;
    }
    free(scratch);
  }
  return res;
}

/* deterministic dot: fixed blocks, partials summed in block order */
static double dot(const double* x, const double* y, int64_t n) {
  const int64_t nb = (n + DOT_BLOCK - 1) / DOT_BLOCK;
  double* part = (double*)malloc(sizeof(double) * (nb > 0 ? nb : 1));
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t lo = b * DOT_BLOCK, hi = lo + DOT_BLOCK < n ? lo + DOT_BLOCK : n;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i) s += x[i] * y[i];
    part[b] = s;
  }
  double t = 0.0;
  for (int64_t b = 0; b < nb; ++b) t += part[b];
  free(part);
  return t;
}

static double norm2(const double* x, int64_t n) { return sqrt(dot(x, x, n)); }

typedef struct {
  const int64_t* rp;
  const int32_t* col;
  const double* val;
  int64_t n;
  double gamma;
  int64_t L;
} Op;

/* y = x - gamma*(P x);  with b: y = b - (x - gamma*(P x)) */
static void apply_J(const Op* op, const double* x, const double* b, double* y) {
#pragma omp parallel
  {
    double* scratch = (double*)malloc(sizeof(double) * op->L);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < op->n; ++r) {
      const double ax = x[r] - op->gamma * row_sum(op->rp, op->col, op->val, x, r, scratch);
      y[r] = b ? b[r] - ax : ax;
    }
    free(scratch);
  }
}

typedef struct {
  int32_t iterations;
  int32_t converged;
  int32_t breakdown;
  int32_t pad;
  double final_resid;
  double eff;
} OrcReport;

static void back_sub(const double* H, const double* g, int j, double* y) {
  for (int i = j - 1; i >= 0; --i) {
    double acc = 0.0;
    for (int k = i + 1; k < j; ++k) acc += H[i * RESTART + k] * y[k];
    const double t = g[i] - acc;
    y[i] = H[i * RESTART + i] != 0.0 ? t / H[i * RESTART + i] : 0.0;
  }
}

/* inner.py:163-292 for kind 0 = richardson, 1 = gmres; x in/out */
int orc_inner_solve(const int64_t* rp, const int32_t* col, const double* val, int64_t n,
                    double gamma, const double* b, double* x, double target, int32_t max_it,
                    int32_t kind, double scale, OrcReport* rep, int nthreads) {
  set_threads(nthreads);
  Op op = {rp, col, val, n, gamma, max_row_len(rp, n) + 1};
  const double bn = norm2(b, n);
  const double eff = fmax(target, 1e-14 * fmax(1.0, bn));
  double* r = (double*)malloc(sizeof(double) * n);
  int it = 0;
  double rn;
  if (kind == 0) {
    for (;;) {
      apply_J(&op, x, b, r);
      rn = norm2(r, n);
      if (rn <= eff || it >= max_it || !isfinite(rn)) break;
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) x[i] = x[i] + scale * r[i];
      ++it;
    }
  } else {
    double* V = (double*)malloc(sizeof(double) * (RESTART + 1) * n);
    double* w = (double*)malloc(sizeof(double) * n);
    double H[(RESTART + 1) * RESTART], cs[RESTART], sn[RESTART], g[RESTART + 1], y[RESTART];
    apply_J(&op, x, b, r);
    rn = norm2(r, n);
    double est = eff;
    while (rn > eff && it < max_it) {
      const double beta = norm2(r, n);
      if (beta == 0.0 || !isfinite(beta)) break;
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) V[i] = r[i] / beta;
      memset(H, 0, sizeof(H));
      memset(cs, 0, sizeof(cs));
      memset(sn, 0, sizeof(sn));
      memset(g, 0, sizeof(g));
      g[0] = beta;
      int j = 0;
      while (j < RESTART && it < max_it) {
        apply_J(&op, V + (int64_t)j * n, NULL, w);
        ++it;
        for (int l = 0; l <= j; ++l) {
          const double* Vl = V + (int64_t)l * n;
          const double h = dot(Vl, w, n);
          H[l * RESTART + j] = h;
#pragma omp parallel for schedule(static)
          for (int64_t i = 0; i < n; ++i) w[i] = w[i] - h * Vl[i];
        }
        const double hn = norm2(w, n);
        H[(j + 1) * RESTART + j] = hn;
        for (int l = 0; l < j; ++l) {
          const double t = cs[l] * H[l * RESTART + j] + sn[l] * H[(l + 1) * RESTART + j];
          H[(l + 1) * RESTART + j] = -sn[l] * H[l * RESTART + j] + cs[l] * H[(l + 1) * RESTART + j];
          H[l * RESTART + j] = t;
        }
        const double denom = hypot(H[j * RESTART + j], H[(j + 1) * RESTART + j]);
        if (denom == 0.0) break;
        cs[j] = H[j * RESTART + j] / denom;
        sn[j] = H[(j + 1) * RESTART + j] / denom;
        H[j * RESTART + j] = denom;
        H[(j + 1) * RESTART + j] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        ++j;
        if (fabs(g[j]) <= est || hn == 0.0) break;
        double* Vn = V + (int64_t)j * n;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) Vn[i] = w[i] / hn;
      }
      if (j == 0) break;
      back_sub(H, g, j, y);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) {
        double t = 0.0;
        for (int l = 0; l < j; ++l) t += V[(int64_t)l * n + i] * y[l];
        x[i] = x[i] + t;
      }
      apply_J(&op, x, b, r);
      rn = norm2(r, n);
      if (rn > eff && fabs(g[j]) <= est) {
        if (fabs(g[j]) == 0.0) break;
        est = fabs(g[j]) * (eff / rn) * 0.5;
      }
    }
    free(V);
    free(w);
  }
  free(r);
  rep->iterations = it;
  rep->final_resid = rn;
  rep->eff = eff;
  rep->converged = rn <= eff;
  rep->breakdown = 0;
  return 0;
}

typedef struct {
  int32_t status; /* 0 converged, 1 outer_cap, 2 stalled */
  int32_t outer;
  int64_t inner;
} OrcStats;

/* driver.py:109-209; v in/out; pi out (int64); hist capacity >= max_outer+1 */
int orc_solve(int64_t n, int32_t m, const int64_t* rp, const int32_t* col, const double* val,
              const double* cost, double gamma, int maximize, double tol, double alpha,
              int32_t max_outer, int32_t max_inner, int32_t kind, int32_t ksp_max_it,
              double scale, double* v, int64_t* pi, double* hist, int32_t hist_cap,
              OrcStats* st, int nthreads) {
  set_threads(nthreads);
  double* applied = (double*)malloc(sizeof(double) * n);
  double* gpi = (double*)malloc(sizeof(double) * n);
  int64_t* rpp = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  const int64_t Lmax = max_row_len(rp, n * m);
  int32_t* colp = (int32_t*)malloc(sizeof(int32_t) * (Lmax * n + 1));
  double* valp = (double*)malloc(sizeof(double) * (Lmax * n + 1));
  int64_t inner_total = 0;
  int stall = 0, k = 0, status = 0;
  for (;;) {
    const double res = orc_greedy(n, m, rp, col, val, cost, gamma, maximize, v, 0, pi, applied,
                                  nthreads);
    if (k < hist_cap) hist[k] = res;
    if (res <= tol) { status = 0; break; }
    if (k >= max_outer) { status = 1; break; }
    if (k > 0 && res >= hist[k - 1]) {
      if (++stall >= 50) { status = 2; break; }
    } else {
      stall = 0;
    }
    rpp[0] = 0;
    for (int64_t s = 0; s < n; ++s) {
      const int64_t r = s * m + pi[s];
      rpp[s + 1] = rpp[s] + (rp[r + 1] - rp[r]);
      gpi[s] = cost[r];
    }
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < n; ++s) {
      const int64_t r = s * m + pi[s];
      memcpy(colp + rpp[s], col + rp[r], sizeof(int32_t) * (rp[r + 1] - rp[r]));
      memcpy(valp + rpp[s], val + rp[r], sizeof(double) * (rp[r + 1] - rp[r]));
    }
    double target;
    int cap;
    if (ksp_max_it > 0) { target = 0.0; cap = ksp_max_it; }
    else { target = alpha * res; cap = max_inner; }
    OrcReport rep;
    orc_inner_solve(rpp, colp, valp, n, gamma, gpi, v, target, cap, kind, scale, &rep, nthreads);
    inner_total += rep.iterations;
    ++k;
  }
  st->status = status;
  st->outer = k;
  st->inner = inner_total;
  free(applied);
  free(gpi);
  free(rpp);
  free(colp);
  free(valp);
  return 0;
}

/* ---- Philox4x32-10 + the C2/C5 locality recipe (generators.py) ---------- */
typedef struct { uint32_t x, y, z, w; } U4;

static U4 philox(U4 c, uint32_t k0, uint32_t k1) {
  for (int i = 0; i < 10; ++i) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    U4 o = {(uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1,
            (uint32_t)p0};
    c = o;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* rows of states [state0, state0+n_states): col/val (n_states*m*K), cost (n_states*m) */
void orc_gen_locality(int64_t n, int32_t m, int32_t K, int64_t W, uint64_t seed, int64_t state0,
                      int64_t n_states, int32_t* col, double* val, double* cost, int nthreads) {
  set_threads(nthreads);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma omp parallel
  {
    int32_t* chosen = (int32_t*)malloc(sizeof(int32_t) * K);
    double* e = (double*)malloc(sizeof(double) * K);
#pragma omp for schedule(static)
    for (int64_t lr = 0; lr < n_states * m; ++lr) {
      const int64_t s = state0 + lr / m;
      const uint64_t r = (uint64_t)(s * m + lr % m);
      const int64_t lo = s - W < 0 ? 0 : s - W, hi = s + W > n - 1 ? n - 1 : s + W;
      const unsigned __int128 span = (unsigned __int128)(hi - lo + 1);
      int cnt = 0;
      for (uint32_t t = 0; cnt < K; ++t) {
        const U4 o = philox((U4){t, (uint32_t)r, (uint32_t)(r >> 32), 0xC2C5u}, k0, k1);
        const uint64_t pos = ((uint64_t)o.z << 32) | o.y;
        int32_t c;
        if (o.x < 3865470566u)
          c = (int32_t)(lo + (int64_t)(((unsigned __int128)pos * span) >> 64));
        else
          c = (int32_t)(((unsigned __int128)pos * (unsigned __int128)n) >> 64);
        int fresh = 1;
        for (int j = 0; j < cnt; ++j)
          if (chosen[j] == c) { fresh = 0; break; }
        if (fresh) chosen[cnt++] = c;
      }
      qsort(chosen, K, sizeof(int32_t), cmp_i32);
      double total = 0.0;
      for (int i = 0; i < K; ++i) {
        const U4 o = philox((U4){(uint32_t)i, (uint32_t)r, (uint32_t)(r >> 32), 0xD1D1u}, k0, k1);
        const uint64_t bits = ((uint64_t)o.y << 21) | (o.x >> 11);
        e[i] = -log(((double)bits + 1.0) * 0x1.0p-53);
        total += e[i];
      }
      for (int i = 0; i < K; ++i) {
        col[lr * K + i] = chosen[i];
        val[lr * K + i] = e[i] / total;
      }
      const U4 o = philox((U4){0u, (uint32_t)r, (uint32_t)(r >> 32), 0xC057u}, k0, k1);
      cost[lr] = (double)(((uint64_t)o.y << 21) | (o.x >> 11)) * 0x1.0p-53;
    }
    free(chosen);
    free(e);
  }
}
