/* Internal helpers of the oracle (TEST INFRASTRUCTURE — see oracle.h). */
#ifndef SPL_ORC_INTERNAL_H
#define SPL_ORC_INTERNAL_H
#include <stdint.h>

#include "oracle.h"

/* C[i*ldc+j] (+)= sum_k A(i,k)·B(k,j); A(i,k)=a[i*ars+k*acs], B(k,j)=b[k*brs+j*bcs]. */
void orc_gemm(int64_t M, int64_t N, int64_t K, const double* a, int64_t ars, int64_t acs,
              const double* b, int64_t brs, int64_t bcs, double* c, int64_t ldc, int accumulate);
int orc_threads(void);

#endif
