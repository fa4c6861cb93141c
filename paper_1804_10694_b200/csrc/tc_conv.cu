// tc_conv.cu -- implicit-GEMM convolution on the 3xTF32 tensor-core kernel
// ("sgemm (matrix multiplication used
// to implement convolutions)", the Conv benchmark).
//
// GEMM view: M = output pixels (b, y, x), N = filters f, K = (ky, kx, c).  The
// A operand is never materialised: each pipeline stage is one TMA im2col-mode
// copy of 128 output pixels x BK channels of one filter tap (the tap enters as
// the TMA's im2col offsets, image borders are zero-filled by the TMA bounding
// box).  B = KRSC filters viewed as the K-major F x (R*S*C) matrix.  Split,
// MMA, K_c promotion and epilogue are the GEMM kernel's (tc_gemm.cuh).
#include "tc_gemm.cuh"

namespace tmk {
namespace {

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn get_encode_im2col() {
  static EncodeIm2colFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  }
  return fn;
}

// NHWC tensor {C, W, H, N}; the bounding box of filter-window origins is
// [-pad, W + pad - S] x [-pad, H + pad - R] (lower corner -pad, upper corner
// pad - (S-1) / pad - (R-1)), so one im2col column walks output pixels in
// (x, y, b) order; a box is 128 pixels x bk channels.
bool encode_im2col(CUtensorMap* map, const ConvArgs& a, int bk, CUtensorMapSwizzle swz) {
  auto enc = get_encode_im2col();
  if (!enc) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(a.c), static_cast<cuuint64_t>(a.w), static_cast<cuuint64_t>(a.h),
                        static_cast<cuuint64_t>(a.nb)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(a.c) * 4, static_cast<cuuint64_t>(a.c * a.w) * 4,
                           static_cast<cuuint64_t>(a.c * a.w * a.h) * 4};
  int lower[2] = {static_cast<int>(-a.pad), static_cast<int>(-a.pad)};                       // {W, H}
  int upper[2] = {static_cast<int>(a.pad - (a.s - 1)), static_cast<int>(a.pad - (a.r - 1))};  // {W, H}
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(a.X), dims, strides, lower, upper,
                   static_cast<cuuint32_t>(bk), static_cast<cuuint32_t>(kBMCta), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int CG, int BN_CTA, int BK>
tm_status launch_conv_cfg(const ConvArgs& a, bool streamk, int num_sms, cudaStream_t stream) {
  using Cfg = TcCfg<CG, BN_CTA, kPrecTf32x3, BK>;
  const CUtensorMapSwizzle swz = BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  CUtensorMap tmA, tmB;
  if (!encode_im2col(&tmA, a, BK, swz)) return TM_ERR_INTERNAL;
  const int64_t K = a.r * a.s * a.c;
  if (!encode_2d(&tmB, a.Wt, a.f, K, K, BK, BN_CTA, swz)) return TM_ERR_INTERNAL;
  const int64_t M = a.nb * a.ho() * a.wo();
  TcParams p{};
  p.A = nullptr;
  p.lda = 0;
  p.m = static_cast<int>(M);
  p.n = static_cast<int>(a.f);
  p.k = static_cast<int>(K);
  p.tiles_m = static_cast<int>((M + Cfg::kTileM - 1) / Cfg::kTileM);
  p.tiles_n = static_cast<int>((a.f + Cfg::kTileN - 1) / Cfg::kTileN);
  p.num_tiles = p.tiles_m * p.tiles_n;
  p.kblocks = static_cast<int>(K / BK);  // C % BK == 0: whole taps x channel chunks
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.C = a.Y;
  p.ldc = a.f;
  p.cv_ho = static_cast<int>(a.ho());
  p.cv_wo = static_cast<int>(a.wo());
  p.cv_s = static_cast<int>(a.s);
  p.cv_c = static_cast<int>(a.c);
  p.cv_pad = static_cast<int>(a.pad);
  return launch_kernel<CG, BN_CTA, kPrecTf32x3, false, true, BK, true>(tmA, tmB, p, num_sms, streamk, stream);
}

}  // namespace

tm_status launch_conv_tc(const ConvArgs& a, int cg, int bn, int bk, bool streamk, int num_sms, cudaStream_t s) {
  if (a.nb * a.ho() * a.wo() > INT32_MAX / 2 || a.r * a.s * a.c > INT32_MAX / 2) return TM_ERR_INVALID_VALUE;
  if (bk == 16) {
    if (cg == 1 && bn == 16) return launch_conv_cfg<1, 16, 16>(a, streamk, num_sms, s);
    if (cg == 1 && bn == 32) return launch_conv_cfg<1, 32, 16>(a, streamk, num_sms, s);
    if (cg == 1 && bn == 64) return launch_conv_cfg<1, 64, 16>(a, streamk, num_sms, s);
    if (cg == 2 && bn == 64) return launch_conv_cfg<2, 64, 16>(a, streamk, num_sms, s);
  } else if (bk == 32) {
    if (cg == 1 && bn == 16) return launch_conv_cfg<1, 16, 32>(a, streamk, num_sms, s);
    if (cg == 1 && bn == 32) return launch_conv_cfg<1, 32, 32>(a, streamk, num_sms, s);
    if (cg == 1 && bn == 64) return launch_conv_cfg<1, 64, 32>(a, streamk, num_sms, s);
    if (cg == 2 && bn == 64) return launch_conv_cfg<2, 64, 32>(a, streamk, num_sms, s);
    if (cg == 2 && bn == 128) return launch_conv_cfg<2, 128, 32>(a, streamk, num_sms, s);
  }
  return TM_ERR_INVALID_VALUE;
}

}  // namespace tmk
