/*
 * oracle/legendre.c -- CPU restatement of the reference's Legendre stage.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the CPU baseline -- never as the product path.
 *
 * Restates /root/reference/pkg/src/sphwav/sht.py:
 *   recursion coefficients a_lm, b_lm ............ sht.py:140-154
 *   normalised Legendre rows with CS phase ........ sht.py:157-187
 *   synthesis accumulation (blocked, sqrt(L)) ..... sht.py:243-261
 *   analysis ring contraction (pairwise sum) ...... sht.py:320-346
 * with ONE deliberate difference: the reference flushes sectoral seeds below
 * 1e-280 to zero (sht.py:179-184), which is wrong above L ~ 1600 (SURVEY.md
 * finding 2).  Here each ring carries an extended exponent (value = p * 2^E,
 * E a multiple of 300) until the value exceeds 2^-700, so the recursion is
 * valid to L = 16383.  Thresholds and seeds are chosen independently of the
 * CUDA kernels (which use 2^256 steps and a 2^-600 switch).
 *
 * Layouts: complex values interleaved (re, im); flm flat l*l + l + m; G
 * ring-major [set][t][bin] with bin = m (m >= 0) or N + m (m < 0), N = 2L-1
 * for complex sets; bins 0..L-1 for real sets.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_STEP 300
#define OR_SWITCH (-700)

typedef struct {
  double p1, p2;
  int E; /* 0: plain value; < 0: scaled by 2^E */
} ring_t;

/* c_m = 1/sqrt(4 pi) prod_{k<=m} sqrt((2k+1)/(2k)) in long double */
static double* seed_table(int L) {
  double* c = (double*)malloc(sizeof(double) * (L > 0 ? L : 1));
  long double v = 1.0L / sqrtl(4.0L * 3.141592653589793238462643383279502884L);
  c[0] = (double)v;
  for (int m = 1; m < L; ++m) {
    v *= sqrtl((long double)(2 * m + 1) / (long double)(2 * m));
    c[m] = (double)v;
  }
  return c;
}

/* (-1)^m c_m s^m  ->  ring state (p2 slot holds the seed, p1 = 0) */
static void ring_seed(ring_t* r, double s, int m, double cm) {
  r->p1 = 0.0;
  r->p2 = 0.0;
  r->E = 0;
  if (m == 0) {
    r->p2 = cm;
    return;
  }
  if (s == 0.0) return;
  /* log2 |seed| split as integer exponent + mantissa via frexp products */
  int e;
  double mant = frexp(cm, &e);
  long long X = e;
  double b = frexp(fabs(s), &e);
  long long be = e;
  for (int n = m; n; n >>= 1) {
    if (n & 1) {
      mant = frexp(mant * b, &e);
      X += be + e;
    }
    if (n > 1) {
      b = frexp(b * b, &e);
      be = 2 * be + e;
    }
  }
  int sign = (m & 1) ? -1 : 1;
  if (s < 0.0 && (m & 1)) sign = -sign;
  if (X > OR_SWITCH) {
    r->p2 = sign * ldexp(mant, (int)X);
  } else {
    long long q = (-X + OR_STEP - 1) / OR_STEP; /* E = -q*STEP <= X */
    r->E = (int)(-q * OR_STEP);
    r->p2 = sign * ldexp(mant, (int)(X - r->E));
  }
}

static inline double ring_next(ring_t* r, double a, double b, double x) {
  double p = a * (x * r->p1) - b * r->p2;
  r->p2 = r->p1;
  r->p1 = p;
  if (r->E < 0) {
    double mx = fmax(fabs(r->p1), fabs(r->p2));
    if (mx > 0x1p300) {
      r->p1 = ldexp(r->p1, -OR_STEP);
      r->p2 = ldexp(r->p2, -OR_STEP);
      r->E += OR_STEP;
      mx = ldexp(mx, -OR_STEP);
    }
    if (mx > 0.0 && r->E + ilogb(mx) > OR_SWITCH) {
      r->p1 = ldexp(r->p1, r->E);
      r->p2 = ldexp(r->p2, r->E);
      r->E = 0;
    }
    return 0.0; /* not yet significant */
  }
  return p;
}

/* sht.py:146-152 operation order */
static inline void rec_ab(int l, int m, double* a, double* b) {
  if (l == m) {
    *a = 0.0;
    *b = -1.0;
    return;
  }
  double L_ = l, M_ = m;
  *a = sqrt((4.0 * L_ * L_ - 1.0) / (L_ * L_ - M_ * M_));
  *b = sqrt((2.0 * L_ + 1.0) / (2.0 * L_ - 3.0) * ((L_ - 1.0) * (L_ - 1.0) - M_ * M_) /
            (L_ * L_ - M_ * M_));
}

/* table[l*L + m] = P_lm(theta) (0 <= m <= l < L) */
void or_legendre_table(int L, double ct, double st, double* table) {
  double* c = seed_table(L);
  memset(table, 0, sizeof(double) * (size_t)L * L);
  for (int m = 0; m < L; ++m) {
    ring_t r;
    ring_seed(&r, st, m, c[m]);
    for (int l = m; l < L; ++l) {
      double a, b;
      rec_ab(l, m, &a, &b);
      (void)ring_next(&r, a, b, ct);
      table[(size_t)l * L + m] = (r.E == 0) ? r.p1 : ldexp(r.p1, r.E);
    }
  }
  free(c);
}

static int resolve_orders(int L, int n_orders, const int* orders, int** out) {
  int* o = (int*)malloc(sizeof(int) * (n_orders > 0 ? n_orders : L));
  if (n_orders > 0) {
    memcpy(o, orders, sizeof(int) * n_orders);
  } else {
    for (int m = 0; m < L; ++m) o[m] = m;
    n_orders = L;
  }
  *out = o;
  return n_orders;
}

/*
 * Synthesis Legendre stage (sht.py:243-261): for every listed order m >= 0
 * and ring t, G_{+m}(t) = sum_l f_lm P_lm(t) and (complex sets)
 * G_{-m}(t) = (-1)^m sum_l f_{l,-m} P_lm(t).  Degrees accumulate in blocks of
 * max(8, floor(sqrt(L))) that are flushed into the total (sht.py:245).
 * n_orders = 0 means all orders 0..L-1.
 */
void or_legendre_synth(int L, int nt, const double* ct, const double* st, int n_sets, int Lc,
                       int real, const double* flm, double* G, int n_orders, const int* orders) {
  const int N = 2 * L - 1, nb = real ? L : N;
  const int flush = (int)fmax(8.0, floor(sqrt((double)L)));
  double* c = seed_table(L);
  int* ord;
  n_orders = resolve_orders(L, n_orders, orders, &ord);
#pragma omp parallel
  {
    ring_t* rs = (ring_t*)malloc(sizeof(ring_t) * nt);
    double* pv = (double*)malloc(sizeof(double) * nt);
    double* acc = (double*)malloc(sizeof(double) * (size_t)nt * n_sets * 4);
    double* tot = (double*)malloc(sizeof(double) * (size_t)nt * n_sets * 4);
#pragma omp for schedule(dynamic, 1)
    for (int oi = 0; oi < n_orders; ++oi) {
      const int m = ord[oi];
      const double sgn = (m & 1) ? -1.0 : 1.0;
      for (int t = 0; t < nt; ++t) ring_seed(&rs[t], st[t], m, c[m]);
      memset(acc, 0, sizeof(double) * (size_t)nt * n_sets * 4);
      memset(tot, 0, sizeof(double) * (size_t)nt * n_sets * 4);
      for (int l = m; l < L; ++l) {
        double a, b;
        rec_ab(l, m, &a, &b);
        for (int t = 0; t < nt; ++t) pv[t] = ring_next(&rs[t], a, b, ct[t]);
        if (l < Lc) {
          for (int s = 0; s < n_sets; ++s) {
            const double* f = flm + 2 * ((size_t)s * Lc * Lc);
            const double fr = f[2 * ((size_t)l * l + l + m)], fi = f[2 * ((size_t)l * l + l + m) + 1];
            double gr = 0, gi = 0;
            if (!real && m > 0) {
              gr = sgn * f[2 * ((size_t)l * l + l - m)];
              gi = sgn * f[2 * ((size_t)l * l + l - m) + 1];
            }
            double* A = acc + (size_t)s * nt * 4;
            for (int t = 0; t < nt; ++t) {
              A[4 * t + 0] += fr * pv[t];
              A[4 * t + 1] += fi * pv[t];
              A[4 * t + 2] += gr * pv[t];
              A[4 * t + 3] += gi * pv[t];
            }
          }
        }
        if ((l + 1) % flush == 0 || l == L - 1) {
          for (size_t i = 0; i < (size_t)nt * n_sets * 4; ++i) {
            tot[i] += acc[i];
            acc[i] = 0.0;
          }
        }
      }
      for (int s = 0; s < n_sets; ++s) {
        const double* T = tot + (size_t)s * nt * 4;
        double* g = G + 2 * ((size_t)s * nt * nb);
        for (int t = 0; t < nt; ++t) {
          g[2 * ((size_t)t * nb + m)] = T[4 * t];
          g[2 * ((size_t)t * nb + m) + 1] = T[4 * t + 1];
          if (!real && m > 0) {
            g[2 * ((size_t)t * nb + N - m)] = T[4 * t + 2];
            g[2 * ((size_t)t * nb + N - m) + 1] = T[4 * t + 3];
          }
        }
      }
    }
    free(rs);
    free(pv);
    free(acc);
    free(tot);
  }
  free(ord);
  free(c);
}

/* pairwise sum of x[0..n) (numpy's reduction shape, sht.py:317-319) */
static double pairwise(const double* x, int n) {
  if (n <= 8) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i];
    return s;
  }
  int h = n / 2;
  return pairwise(x, h) + pairwise(x + h, n - h);
}

/*
 * Analysis Legendre stage (sht.py:320-346): f_lm = sum_t P_lm(t) w_t H_m(t),
 * rings reduced pairwise.  H is m-major [set][bin][t] (bins as in
 * or_legendre_synth); w_t includes every normalisation.  Complex sets also
 * produce f_{l,-m} = (-1)^m sum_t P_lm w_t H_{-m}; real sets mirror
 * f_{l,-m} = (-1)^m conj f_lm exactly (sht.py:328-331) and keep f_l0 real.
 * Output flm [set][L*L] is written only at the listed orders.
 */
void or_legendre_ana(int L, int nt, const double* ct, const double* st, const double* w,
                     int n_sets, int real, const double* H, double* flm, int n_orders,
                     const int* orders) {
  const int N = 2 * L - 1, nb = real ? L : N;
  double* c = seed_table(L);
  int* ord;
  n_orders = resolve_orders(L, n_orders, orders, &ord);
#pragma omp parallel
  {
    ring_t* rs = (ring_t*)malloc(sizeof(ring_t) * nt);
    double* pv = (double*)malloc(sizeof(double) * nt);
    double* tmp = (double*)malloc(sizeof(double) * nt);
    double* hw = (double*)malloc(sizeof(double) * (size_t)nt * n_sets * 4);
#pragma omp for schedule(dynamic, 1)
    for (int oi = 0; oi < n_orders; ++oi) {
      const int m = ord[oi];
      const double sgn = (m & 1) ? -1.0 : 1.0;
      for (int s = 0; s < n_sets; ++s) {
        const double* h = H + 2 * ((size_t)s * nb * nt);
        for (int t = 0; t < nt; ++t) {
          double* q = hw + ((size_t)s * 4) * nt;
          q[t] = h[2 * ((size_t)m * nt + t)] * w[t];
          q[nt + t] = h[2 * ((size_t)m * nt + t) + 1] * w[t];
          q[2 * nt + t] = (!real && m > 0) ? h[2 * ((size_t)(N - m) * nt + t)] * w[t] : 0.0;
          q[3 * nt + t] = (!real && m > 0) ? h[2 * ((size_t)(N - m) * nt + t) + 1] * w[t] : 0.0;
        }
      }
      for (int t = 0; t < nt; ++t) ring_seed(&rs[t], st[t], m, c[m]);
      for (int l = m; l < L; ++l) {
        double a, b;
        rec_ab(l, m, &a, &b);
        for (int t = 0; t < nt; ++t) pv[t] = ring_next(&rs[t], a, b, ct[t]);
        for (int s = 0; s < n_sets; ++s) {
          double v[4];
          for (int k = 0; k < 4; ++k) {
            const double* q = hw + ((size_t)s * 4 + k) * nt;
            for (int t = 0; t < nt; ++t) tmp[t] = pv[t] * q[t];
            v[k] = pairwise(tmp, nt);
          }
          double* f = flm + 2 * ((size_t)s * L * L);
          const size_t ip = (size_t)l * l + l + m, im = (size_t)l * l + l - m;
          f[2 * ip] = v[0];
          f[2 * ip + 1] = (real && m == 0) ? 0.0 : v[1];
          if (m > 0) {
            if (real) {
              f[2 * im] = sgn * v[0];
              f[2 * im + 1] = -sgn * v[1];
            } else {
              f[2 * im] = sgn * v[2];
              f[2 * im + 1] = sgn * v[3];
            }
          }
        }
      }
    }
    free(rs);
    free(pv);
    free(tmp);
    free(hw);
  }
  free(ord);
  free(c);
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
