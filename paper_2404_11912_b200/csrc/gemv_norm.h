// Folded-RMSNorm parameters of the tensor-core GEMV (gemv_tc.cu), used by
// the single-row-block forward (forward.cu): norms never run as separate
// kernels -- the residual-producing GEMV writes the next operand split(x * g);
// the consuming GEMV computes 1 / rms(x) from x while its weights stream and
// scales its result by it.
#pragma once

#include <stdint.h>

namespace hs {

struct GemvNorm {
  const float *x_in;      // consumer: the un-normalised input rows [t][ldx_in] (null: no norm)
  int ldx_in, norm_K;     // row stride; K of the mean
  float eps;
  const float *gnext;     // producer: gain of the next norm
  uint16_t *xs_next;      // producer: next operand [24][ld_next] (null: none)
  int ld_next;
};

}  // namespace hs
