/*
 * s2w_testing.h -- stage-level hooks of libs2w.so used by the parity tests.
 * Not part of the drop-in surface (include/s2w.h); same kernels, one stage at
 * a time, device pointers, asynchronous on `stream`.
 */
#ifndef S2W_TESTING_H
#define S2W_TESTING_H
#ifdef __cplusplus
extern "C" {
#endif
/* G ring-major [set][t][bin] (bins: 2L-1 complex / L real) -> map rows
 * (inverse ring DFT, unnormalised; MW pole pinning). */
int s2w_test_rings_inverse(int scheme, int L, int n_sets, int is_real, const double* G,
                           double* map, void* stream);
/* map rows -> G m-major [set][bin][t] = DFT/N; theta_stage != 0 also applies the
 * MW theta stage (the symmetrised H of DESIGN.md). */
int s2w_test_rings_forward(int scheme, int L, int n_sets, int is_real, int theta_stage,
                           const double* map, double* G, void* stream);
#ifdef __cplusplus
}
#endif
#endif
