/* oracle/legendre_body.h -- the generic body of legendre.c, instantiated for
 * R = double (the reference's arithmetic) and R = long double (the precise
 * checker).  TEST INFRASTRUCTURE ONLY; see legendre.c. */
typedef struct {
  R p1, p2;
  int E; /* 0: plain value; < 0: scaled by 2^E */
} SFX(ring_t);

/* c_m = 1/sqrt(4 pi) prod_{k<=m} sqrt((2k+1)/(2k)) in long double */
static R* SFX(seed_table)(int L) {
  R* c = (R*)malloc(sizeof(R) * (L > 0 ? L : 1));
  long double v = 1.0L / sqrtl(4.0L * 3.141592653589793238462643383279502884L);
  c[0] = (R)v;
  for (int m = 1; m < L; ++m) {
    v *= sqrtl((long double)(2 * m + 1) / (long double)(2 * m));
    c[m] = (R)v;
  }
  return c;
}

/* (-1)^m c_m s^m  ->  ring state (p2 slot holds the seed, p1 = 0) */
static void SFX(ring_seed)(SFX(ring_t) * r, R s, int m, R cm) {
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
  R mant = M(frexp)(cm, &e);
  long long X = e;
  R b = M(frexp)(M(fabs)(s), &e);
  long long be = e;
  for (int n = m; n; n >>= 1) {
    if (n & 1) {
      mant = M(frexp)(mant * b, &e);
      X += be + e;
    }
    if (n > 1) {
      b = M(frexp)(b * b, &e);
      be = 2 * be + e;
    }
  }
  int sign = (m & 1) ? -1 : 1;
  if (s < 0.0 && (m & 1)) sign = -sign;
  if (X > OR_SWITCH) {
    r->p2 = sign * M(ldexp)(mant, (int)X);
  } else {
    long long q = (-X + OR_STEP - 1) / OR_STEP; /* E = -q*STEP <= X */
    r->E = (int)(-q * OR_STEP);
    r->p2 = sign * M(ldexp)(mant, (int)(X - r->E));
  }
}

/* x * p with the exact node when cd != 0 (see the header) */
static inline R SFX(xmul)(R x, R cd, R p) {
  if (cd == 0.0) return x * p;
  return x > 0.0 ? p - cd * p : cd * p - p;
}

static inline R SFX(ring_next)(SFX(ring_t) * r, R a, R b, R x, R cd) {
  R p = a * SFX(xmul)(x, cd, r->p1) - b * r->p2;
  r->p2 = r->p1;
  r->p1 = p;
  if (r->E < 0) {
    R mx = M(fmax)(M(fabs)(r->p1), M(fabs)(r->p2));
    if (mx > 0x1p300) {
      r->p1 = M(ldexp)(r->p1, -OR_STEP);
      r->p2 = M(ldexp)(r->p2, -OR_STEP);
      r->E += OR_STEP;
      mx = M(ldexp)(mx, -OR_STEP);
    }
    if (mx > 0.0 && r->E + M(ilogb)(mx) > OR_SWITCH) {
      r->p1 = M(ldexp)(r->p1, r->E);
      r->p2 = M(ldexp)(r->p2, r->E);
      r->E = 0;
    }
    return 0.0; /* not yet significant */
  }
  return p;
}

/* sht.py:146-152 operation order */
static inline void SFX(rec_ab)(int l, int m, R* a, R* b) {
  if (l == m) {
    *a = 0.0;
    *b = -1.0;
    return;
  }
  R L_ = l, M_ = m;
  *a = M(sqrt)((4.0 * L_ * L_ - 1.0) / (L_ * L_ - M_ * M_));
  *b = M(sqrt)((2.0 * L_ + 1.0) / (2.0 * L_ - 3.0) * ((L_ - 1.0) * (L_ - 1.0) - M_ * M_) /
               (L_ * L_ - M_ * M_));
}

/* table[l*L + m] = P_lm(theta) (0 <= m <= l < L) */
static void SFX(table)(int L, R ct, R st, R cd, double* table) {
  R* c = SFX(seed_table)(L);
  memset(table, 0, sizeof(double) * (size_t)L * L);
  for (int m = 0; m < L; ++m) {
    SFX(ring_t) r;
    SFX(ring_seed)(&r, st, m, c[m]);
    for (int l = m; l < L; ++l) {
      R a, b;
      SFX(rec_ab)(l, m, &a, &b);
      (void)SFX(ring_next)(&r, a, b, ct, cd);
      table[(size_t)l * L + m] = (double)((r.E == 0) ? r.p1 : M(ldexp)(r.p1, r.E));
    }
  }
  free(c);
}

static int SFX(resolve_orders)(int L, int n_orders, const int* orders, int** out) {
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
static void SFX(synth)(int L, int nt, const double* ct, const double* st, const double* cd,
                       int n_sets, int Lc, int real, const double* flm, double* G, int n_orders,
                       const int* orders) {
  const int N = 2 * L - 1, nb = real ? L : N;
  const int flush = (int)fmax(8.0, floor(sqrt((double)L)));
  R* c = SFX(seed_table)(L);
  int* ord;
  n_orders = SFX(resolve_orders)(L, n_orders, orders, &ord);
#pragma omp parallel
  {
    SFX(ring_t)* rs = (SFX(ring_t)*)malloc(sizeof(SFX(ring_t)) * nt);
    R* pv = (R*)malloc(sizeof(R) * nt);
    R* acc = (R*)malloc(sizeof(R) * (size_t)nt * n_sets * 4);
    R* tot = (R*)malloc(sizeof(R) * (size_t)nt * n_sets * 4);
#pragma omp for schedule(dynamic, 1)
    for (int oi = 0; oi < n_orders; ++oi) {
      const int m = ord[oi];
      const R sgn = (m & 1) ? -1.0 : 1.0;
      for (int t = 0; t < nt; ++t) SFX(ring_seed)(&rs[t], st[t], m, c[m]);
      memset(acc, 0, sizeof(R) * (size_t)nt * n_sets * 4);
      memset(tot, 0, sizeof(R) * (size_t)nt * n_sets * 4);
      for (int l = m; l < L; ++l) {
        R a, b;
        SFX(rec_ab)(l, m, &a, &b);
        for (int t = 0; t < nt; ++t) pv[t] = SFX(ring_next)(&rs[t], a, b, ct[t], cd ? cd[t] : 0.0);
        if (l < Lc) {
          for (int s = 0; s < n_sets; ++s) {
            const double* f = flm + 2 * ((size_t)s * Lc * Lc);
            const R fr = f[2 * ((size_t)l * l + l + m)], fi = f[2 * ((size_t)l * l + l + m) + 1];
            R gr = 0, gi = 0;
            if (!real && m > 0) {
              gr = sgn * f[2 * ((size_t)l * l + l - m)];
              gi = sgn * f[2 * ((size_t)l * l + l - m) + 1];
            }
            R* A = acc + (size_t)s * nt * 4;
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
        const R* T = tot + (size_t)s * nt * 4;
        double* g = G + 2 * ((size_t)s * nt * nb);
        for (int t = 0; t < nt; ++t) {
          g[2 * ((size_t)t * nb + m)] = (double)T[4 * t];
          g[2 * ((size_t)t * nb + m) + 1] = (double)T[4 * t + 1];
          if (!real && m > 0) {
            g[2 * ((size_t)t * nb + N - m)] = (double)T[4 * t + 2];
            g[2 * ((size_t)t * nb + N - m) + 1] = (double)T[4 * t + 3];
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
static R SFX(pairwise)(const R* x, int n) {
  if (n <= 8) {
    R s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i];
    return s;
  }
  int h = n / 2;
  return SFX(pairwise)(x, h) + SFX(pairwise)(x + h, n - h);
}

/*
 * Analysis Legendre stage (sht.py:320-346): f_lm = sum_t P_lm(t) w_t H_m(t),
 * rings reduced pairwise.  H is m-major [set][bin][t] (bins as in
 * or_legendre_synth); w_t includes every normalisation.  Complex sets also
 * produce f_{l,-m} = (-1)^m sum_t P_lm w_t H_{-m}; real sets mirror
 * f_{l,-m} = (-1)^m conj f_lm exactly (sht.py:328-331) and keep f_l0 real.
 * Output flm [set][L*L] is written only at the listed orders.
 */
static void SFX(ana)(int L, int nt, const double* ct, const double* st, const double* cd,
                     const double* w, int n_sets, int real, const double* H, double* flm,
                     int n_orders, const int* orders) {
  const int N = 2 * L - 1, nb = real ? L : N;
  R* c = SFX(seed_table)(L);
  int* ord;
  n_orders = SFX(resolve_orders)(L, n_orders, orders, &ord);
#pragma omp parallel
  {
    SFX(ring_t)* rs = (SFX(ring_t)*)malloc(sizeof(SFX(ring_t)) * nt);
    R* pv = (R*)malloc(sizeof(R) * nt);
    R* tmp = (R*)malloc(sizeof(R) * nt);
    R* hw = (R*)malloc(sizeof(R) * (size_t)nt * n_sets * 4);
#pragma omp for schedule(dynamic, 1)
    for (int oi = 0; oi < n_orders; ++oi) {
      const int m = ord[oi];
      const R sgn = (m & 1) ? -1.0 : 1.0;
      for (int s = 0; s < n_sets; ++s) {
        const double* h = H + 2 * ((size_t)s * nb * nt);
        for (int t = 0; t < nt; ++t) {
          R* q = hw + ((size_t)s * 4) * nt;
          q[t] = (R)h[2 * ((size_t)m * nt + t)] * w[t];
          q[nt + t] = (R)h[2 * ((size_t)m * nt + t) + 1] * w[t];
          q[2 * nt + t] = (!real && m > 0) ? (R)h[2 * ((size_t)(N - m) * nt + t)] * w[t] : 0.0;
          q[3 * nt + t] = (!real && m > 0) ? (R)h[2 * ((size_t)(N - m) * nt + t) + 1] * w[t] : 0.0;
        }
      }
      for (int t = 0; t < nt; ++t) SFX(ring_seed)(&rs[t], st[t], m, c[m]);
      for (int l = m; l < L; ++l) {
        R a, b;
        SFX(rec_ab)(l, m, &a, &b);
        for (int t = 0; t < nt; ++t) pv[t] = SFX(ring_next)(&rs[t], a, b, ct[t], cd ? cd[t] : 0.0);
        for (int s = 0; s < n_sets; ++s) {
          R v[4];
          for (int k = 0; k < 4; ++k) {
            const R* q = hw + ((size_t)s * 4 + k) * nt;
            for (int t = 0; t < nt; ++t) tmp[t] = pv[t] * q[t];
            v[k] = SFX(pairwise)(tmp, nt);
          }
          double* f = flm + 2 * ((size_t)s * L * L);
          const size_t ip = (size_t)l * l + l + m, im = (size_t)l * l + l - m;
          f[2 * ip] = (double)v[0];
          f[2 * ip + 1] = (real && m == 0) ? 0.0 : (double)v[1];
          if (m > 0) {
            if (real) {
              f[2 * im] = (double)(sgn * v[0]);
              f[2 * im + 1] = (double)(-sgn * v[1]);
            } else {
              f[2 * im] = (double)(sgn * v[2]);
              f[2 * im + 1] = (double)(sgn * v[3]);
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

