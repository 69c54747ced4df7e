// Triangle collections (tri.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spechp_b200.h"

namespace sphp {

struct TriJob {
  int op;
  int m1, nm, Q1, Q2;
  int ntab;            // doubles in tab
  const double* tab;   // device: A1 (m1,Q1) | B2 (nm,Q2) | D1 | D2 | f (Q2) | g (Q1*Q2) | w (Q1*Q2)
  const int* itab;     // device: pidx (nm) | bstart (m1+1)
  int geom_kind;       // NONE, AFFINE ([det, inv00, inv01, inv10, inv11]) or POINT ([wJ | inv] planes)
  const double* geom;
  int64_t gstride, cs;
  int64_t E;
  const double* in;
  double* out;
};

size_t tri_smem_bytes(const TriJob& j);
cudaError_t tri_apply(const TriJob& j, int num_sms, cudaStream_t s);

}  // namespace sphp
