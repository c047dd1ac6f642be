// Convolution ops of the training step: forward, data gradient, weight
// gradient.  bf16 activations dispatch to the tcgen05
// tensor-core implicit GEMM (conv_tc.cu) when the shape fits its tiling
// (channels in multiples of 64; the 3-channel stem gathers into registers),
// else to the CUDA-core implicit GEMM (conv_simt.cu).  fp32 activations
// (attrs.dtype = "f32", the 1e-5 parity mode) always run on CUDA cores — no
// TF32.  attrs.impl = "simt" or OC_CONV_IMPL=simt force CUDA cores.
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
bool f32(const OpArgs& a) { return As(a, "dtype", "bf16") == "f32"; }

enum { CF_X, CF_W, CF_Y };
Status conv_fwd(OpArgs& a) {
  ConvGeom g = conv_geom(a);
  auto w = (const float*)a.p(CF_W);
  if (f32(a)) return conv_fprop_simt<float>(a, g, (const float*)a.p(CF_X), w, (float*)a.p(CF_Y));
  auto x = (const __nv_bfloat16*)a.p(CF_X);
  auto y = (__nv_bfloat16*)a.p(CF_Y);
  if (!force_simt(&a) && conv_tc_ok(g, 0)) return conv_fprop_tc(a, g, x, w, y);
  return conv_fprop_simt<__nv_bfloat16>(a, g, x, w, y);
}

enum { CD_DY, CD_W, CD_DX };
Status conv_dgrad(OpArgs& a) {
  ConvGeom g = conv_geom(a);
  auto w = (const float*)a.p(CD_W);
  const bool acc = Ab(a, "accumulate");
  if (f32(a)) return conv_dgrad_simt<float>(a, g, (const float*)a.p(CD_DY), w, (float*)a.p(CD_DX), acc);
  auto dy = (const __nv_bfloat16*)a.p(CD_DY);
  auto dx = (__nv_bfloat16*)a.p(CD_DX);
  if (!force_simt(&a) && conv_tc_ok(g, 1)) return conv_dgrad_tc(a, g, dy, w, dx, acc);
  return conv_dgrad_simt<__nv_bfloat16>(a, g, dy, w, dx, acc);
}

enum { CW_DY, CW_X, CW_DW };
Status conv_wgrad(OpArgs& a) {
  ConvGeom g = conv_geom(a);
  auto dw = (float*)a.p(CW_DW);
  if (f32(a)) return conv_wgrad_simt<float>(a, g, (const float*)a.p(CW_DY), (const float*)a.p(CW_X), dw);
  auto dy = (const __nv_bfloat16*)a.p(CW_DY);
  auto x = (const __nv_bfloat16*)a.p(CW_X);
  if (!force_simt(&a) && conv_tc_ok(g, 2)) return conv_wgrad_tc(a, g, dy, x, dw);
  return conv_wgrad_simt<__nv_bfloat16>(a, g, dy, x, dw);
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
