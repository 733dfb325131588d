// Operand-plane format of the Gram / projection / scaled-matrix planes: BF16 hi/lo, or FP16
// hi = fp16(z), lo = fp16(z - hi) (11-bit significands, the TF32 rounding at the full kind::f16
// rate; needs |z| < 65504, true for scaled data).  Included after <cuda_bf16.h> in the files
// that write or read the planes; under SCB_PLANES_F16 it renames the BF16 intrinsics used there.
#pragma once
// Default: BF16 planes and the three-product Gram.  Build switches (measured):
// -DSCB_PLANES_F16 FP16 planes (no accuracy gain: the FP32 accumulation dominates), plus
// -DSCB_GRAM_1X the one-product (hi x hi) Gram (PCA 15.0 -> 12.8 ms at C3, but subspace angles
// of 1.0-1.7e-3 on the small C1 / edge configurations, over the 1e-3 bar).
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
