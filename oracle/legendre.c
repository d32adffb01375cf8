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
 * Polar rings: the reference multiplies by x = fl(cos theta) (sht.py:172-185).
 * Within |x| > 1/2 of a pole the rounding of x moves the node by up to
 * eps/(1 -/+ x) relative in 1 -/+ x, which at L = 4096 shifts P_l0 on the
 * first MW ring by ~1.2e-10 of its scale (measured against mpmath,
 * tests/test_oracle.py).  The caller may pass cd = 1 - x (x > 1/2) or 1 + x
 * (x < -1/2) computed from the exact node; x * p is then formed as
 * p - cd * p (resp. cd * p - p), i.e. with the exact node.  cd = 0 keeps the
 * reference's product.
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

/* R = double: the reference's arithmetic (the CPU baseline times this one) */
#define R double
#define SFX(x) x##_d
#define M(f) f
#include "legendre_body.h"
#undef R
#undef SFX
#undef M

/* R = long double (x87, 64-bit mantissa): the checker.  The recursion's own
 * rounding near the poles reaches ~1.5e-10 of the P_l scale in double at
 * L = 4096 (pinned against mpmath in tests/test_oracle.py); in long double it
 * is ~2000x smaller, so the checker is accurate well below the 1e-10 bar. */
#define R long double
#define SFX(x) x##_ld
#define M(f) f##l
#include "legendre_body.h"
#undef R
#undef SFX
#undef M

/* precise != 0 selects the long-double instantiation */
void or_legendre_table(int L, double ct, double st, double cd, double* table, int precise) {
  if (precise) table_ld(L, ct, st, cd, table);
  else table_d(L, ct, st, cd, table);
}

void or_legendre_synth(int L, int nt, const double* ct, const double* st, const double* cd,
                       int n_sets, int Lc, int real, const double* flm, double* G, int n_orders,
                       const int* orders, int precise) {
  if (precise) synth_ld(L, nt, ct, st, cd, n_sets, Lc, real, flm, G, n_orders, orders);
  else synth_d(L, nt, ct, st, cd, n_sets, Lc, real, flm, G, n_orders, orders);
}

void or_legendre_ana(int L, int nt, const double* ct, const double* st, const double* cd,
                     const double* w, int n_sets, int real, const double* H, double* flm,
                     int n_orders, const int* orders, int precise) {
  if (precise) ana_ld(L, nt, ct, st, cd, w, n_sets, real, H, flm, n_orders, orders);
  else ana_d(L, nt, ct, st, cd, w, n_sets, real, H, flm, n_orders, orders);
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
