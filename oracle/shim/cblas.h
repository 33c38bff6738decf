/* cblas.h -- minimal CBLAS declarations so the reference's matrix.cpp compiles for the
 * oracle build (OpenBLAS is absent from this image).  TEST INFRASTRUCTURE ONLY: the naive
 * implementation is oracle/cblas_shim.c; nothing on the product path uses it. */
#ifndef TGFX_ORACLE_CBLAS_SHIM_H
#define TGFX_ORACLE_CBLAS_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void cblas_dgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb, int m,
                 int n, int k, double alpha, const double* a, int lda, const double* b, int ldb,
                 double beta, double* c, int ldc);
void openblas_set_num_threads(int n);
#ifdef __cplusplus
}
#endif
#endif
