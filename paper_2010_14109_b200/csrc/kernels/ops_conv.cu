// Convolution ops of the training step: forward, data gradient, weight
// gradient.  Dispatches to the tcgen05 tensor-core
// implicit GEMM (conv_tc.cu) when the shape fits its tiling, else to the
// CUDA-core implicit GEMM (conv_simt.cu).  attrs.impl = "simt" forces the
// latter (cross-checks).
#include "conv.cuh"

namespace oc {

namespace {

enum { CF_X, CF_W, CF_Y };
Status conv_fwd(OpArgs& a) {
  ConvGeom g = conv_geom(a);
  return conv_fprop_simt(a, g, (const __nv_bfloat16*)a.p(CF_X), (const float*)a.p(CF_W), (__nv_bfloat16*)a.p(CF_Y));
}

enum { CD_DY, CD_W, CD_DX };
Status conv_dgrad(OpArgs& a) {
  ConvGeom g = conv_geom(a);
  return conv_dgrad_simt(a, g, (const __nv_bfloat16*)a.p(CD_DY), (const float*)a.p(CD_W), (__nv_bfloat16*)a.p(CD_DX),
                         Ab(a, "accumulate"));
}

enum { CW_DY, CW_X, CW_DW };
Status conv_wgrad(OpArgs& a) {
  ConvGeom g = conv_geom(a);
  return conv_wgrad_simt(a, g, (const __nv_bfloat16*)a.p(CW_DY), (const __nv_bfloat16*)a.p(CW_X), (float*)a.p(CW_DW));
}
size_t conv_wgrad_ws(const JVal& at) { return conv_wgrad_ws_simt(conv_geom(at)); }

}  // namespace

extern const OpDesc kConvFwd{"conv_fwd", {"x", "w", "y"}, conv_fwd, nullptr};
extern const OpDesc kConvDgrad{"conv_dgrad", {"dy", "w", "dx"}, conv_dgrad, nullptr};
extern const OpDesc kConvWgrad{"conv_wgrad", {"dy", "x", "dw"}, conv_wgrad, conv_wgrad_ws};

}  // namespace oc
