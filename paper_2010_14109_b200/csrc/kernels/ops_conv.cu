// Convolution ops of the training step: forward, data gradient, weight
// gradient.  Dispatches to the tcgen05 tensor-core
// implicit GEMM (conv_tc.cu) when the shape fits its tiling (channels in
// multiples of 64; the 3-channel stem stays on CUDA cores), else to the
// CUDA-core implicit GEMM (conv_simt.cu).  attrs.impl = "simt" or the
// environment variable OC_CONV_IMPL=simt force the latter (cross-checks).
#include <cstdlib>
#include <cstring>

#include "conv.cuh"

namespace oc {

bool conv_tc_ok(const ConvGeom& g, int mode);
size_t conv_tc_ws(const ConvGeom& g, int mode);
Status conv_fprop_tc(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* x, const float* w, __nv_bfloat16* y);
Status conv_dgrad_tc(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* dy, const float* w, __nv_bfloat16* dx,
                     bool accumulate);
Status conv_wgrad_tc(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* dy, const __nv_bfloat16* x, float* dw);

namespace {

bool force_simt(const OpArgs* a) {
  static int env = -1;
  if (env < 0) {
    const char* e = std::getenv("OC_CONV_IMPL");
    env = (e && std::strcmp(e, "simt") == 0) ? 1 : 0;
  }
  return env == 1 || (a && As(*a, "impl") == "simt");
}

enum { CF_X, CF_W, CF_Y };
Status conv_fwd(OpArgs& a) {
  ConvGeom g = conv_geom(a);
  auto x = (const __nv_bfloat16*)a.p(CF_X);
  auto w = (const float*)a.p(CF_W);
  auto y = (__nv_bfloat16*)a.p(CF_Y);
  if (!force_simt(&a) && conv_tc_ok(g, 0)) return conv_fprop_tc(a, g, x, w, y);
  return conv_fprop_simt(a, g, x, w, y);
}

enum { CD_DY, CD_W, CD_DX };
Status conv_dgrad(OpArgs& a) {
  ConvGeom g = conv_geom(a);
  auto dy = (const __nv_bfloat16*)a.p(CD_DY);
  auto w = (const float*)a.p(CD_W);
  auto dx = (__nv_bfloat16*)a.p(CD_DX);
  if (!force_simt(&a) && conv_tc_ok(g, 1)) return conv_dgrad_tc(a, g, dy, w, dx, Ab(a, "accumulate"));
  return conv_dgrad_simt(a, g, dy, w, dx, Ab(a, "accumulate"));
}

enum { CW_DY, CW_X, CW_DW };
Status conv_wgrad(OpArgs& a) {
  ConvGeom g = conv_geom(a);
  auto dy = (const __nv_bfloat16*)a.p(CW_DY);
  auto x = (const __nv_bfloat16*)a.p(CW_X);
  auto dw = (float*)a.p(CW_DW);
  if (!force_simt(&a) && conv_tc_ok(g, 2)) return conv_wgrad_tc(a, g, dy, x, dw);
  return conv_wgrad_simt(a, g, dy, x, dw);
}

size_t ws_fwd(const JVal& at) { return conv_tc_ws(conv_geom(at), 0); }
size_t ws_dgrad(const JVal& at) { return conv_tc_ws(conv_geom(at), 1); }
size_t ws_wgrad(const JVal& at) {
  ConvGeom g = conv_geom(at);
  return std::max(conv_wgrad_ws_simt(g), conv_tc_ws(g, 2));
}

}  // namespace

extern const OpDesc kConvFwd{"conv_fwd", {"x", "w", "y"}, conv_fwd, ws_fwd};
extern const OpDesc kConvDgrad{"conv_dgrad", {"dy", "w", "dx"}, conv_dgrad, ws_dgrad};
extern const OpDesc kConvWgrad{"conv_wgrad", {"dy", "x", "dw"}, conv_wgrad, ws_wgrad};

}  // namespace oc
