/* cblas_shim.c -- naive row-major dgemm for the oracle build of the reference's matrix.cpp
 * (TEST INFRASTRUCTURE ONLY; see oracle/shim/cblas.h). */
#include "shim/cblas.h"

void cblas_dgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb, int m,
                 int n, int k, double alpha, const double* a, int lda, const double* b, int ldb,
                 double beta, double* c, int ldc) {
  (void)order; /* the reference only calls row-major */
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int p = 0; p < k; ++p) {
        const double x = ta == CblasNoTrans ? a[i * lda + p] : a[p * lda + i];
        const double y = tb == CblasNoTrans ? b[p * ldb + j] : b[j * ldb + p];
        s += x * y;
      }
      c[i * ldc + j] = alpha * s + (beta == 0.0 ? 0.0 : beta * c[i * ldc + j]);
    }
}

void openblas_set_num_threads(int n) { (void)n; }
