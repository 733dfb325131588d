// Operand-plane format of the Gram / projection / scaled-matrix planes.  Default BF16 hi/lo.
// Experiment switch SCB_PLANES_F16: FP16 hi = fp16(z), lo = fp16(z - hi) instead (11-bit
// significands: ~2^-22 per 3-product term, the 3xTF32 figure, at the same kind::f16 rate;
// needs |z| < 65504, true for scaled and clipped data).  Included after <cuda_bf16.h> in the
// files that write or read the planes; it renames the BF16 intrinsics used there.
#pragma once
#ifdef SCB_PLANES_F16
#include <cuda_fp16.h>
#define __nv_bfloat16 __half
#define __nv_bfloat162 __half2
#define __floats2bfloat162_rn __floats2half2_rn
#define __bfloat1622float2 __half22float2
#define __float2bfloat16_rn __float2half_rn
#define __bfloat162float __half2float
#define SCB_PLANES_IDESC idesc_f16
#else
#define SCB_PLANES_IDESC idesc_bf16
#endif
