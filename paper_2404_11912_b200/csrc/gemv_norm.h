// Folded-RMSNorm parameters of the tensor-core GEMV (gemv_tc.cu), used by
// the single-row-block forward (forward.cu): norms never run as separate
// kernels -- the residual-producing GEMV writes the next operand split(x * g)
// and per-tile row sums of squares; the consuming GEMV scales by 1 / rms.
#pragma once

#include <stdint.h>

namespace hs {

struct GemvNorm {
  const double *ssq_in;   // consumer: [ssq_parts][8] row sums of squares of its input (null: none)
  int ssq_parts, norm_K;  // parts to sum; K of the mean
  float eps;
  const float *gnext;     // producer: gain of the next norm
  uint16_t *xs_next;      // producer: next operand [24][ld_next] (null: none)
  int ld_next;
  double *ssq_out;        // producer: [tiles][8]
};

}  // namespace hs
