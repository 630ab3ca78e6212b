// host_math.h -- fp64 host steps of the hot path (see host_math.cpp).
#pragma once

namespace ciqh {
// K(m) with the complementary parameter m1 = 1 - m supplied exactly.
double ellipk_comp(double m, double m1);
// Jacobi sn, cn, dn (u | m), complementary parameter m1 = 1 - m supplied exactly.
void ellipj_comp(double u, double m, double m1, double* sn, double* cn, double* dn);
// HHT shifts/weights. 0 ok, -1 bad args, -2 non-finite / non-positive output.
int hht_rule(double lambda_min, double lambda_max, int Q, double* t, double* w);
// Extreme eigenvalues of a symmetric tridiagonal matrix (Sturm bisection). 0 ok.
int tridiag_extremes(const double* alpha, const double* beta, int m, double* emin, double* emax);
// Symmetric eigendecomposition (cyclic Jacobi, fp64): w descending, eigenvectors in columns of v.
int sym_eig_jacobi(double* a, int n, double* w, double* v);
}  // namespace ciqh
